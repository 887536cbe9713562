import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1707_02000_b200 import graphgen, trussdec
from oracle import Oracle, Reference
cfg = int(sys.argv[1])
n, m, off, nb = graphgen.config(cfg)
src = np.repeat(np.arange(n, dtype=np.int64), np.diff(off))
up = src < nb
pairs = np.stack([src[up], nb[up].astype(np.int64)], 1)
rng = np.random.default_rng(1)
pairs = pairs[rng.permutation(len(pairs))]
flip = rng.random(len(pairs)) < 0.5
pairs[flip] = pairs[flip][:, ::-1]
pairs = np.ascontiguousarray(pairs)
gc = trussdec.canonicalize(pairs.astype(np.uint64))
rc = Reference().make_graph(2, 0, 0.0, 0, pairs=pairs)
oc = Oracle().canonicalize(pairs.astype(np.uint64))
for name, x in (("ref", rc), ("oracle", oc)):
    print(name, gc.n, x.n, gc.m, x.m, gc.n == x.n and bool((gc.offsets == x.offsets).all()),
          gc.m == x.m and bool((gc.neighbors == x.neighbors).all()), flush=True)
print("ref==oracle", rc.n == oc.n and bool((rc.offsets == oc.offsets).all()) and bool((rc.neighbors == oc.neighbors).all()))
