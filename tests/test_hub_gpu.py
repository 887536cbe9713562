"""GPU: the support pass's HUB path — owners whose oriented list exceeds one shared-memory
table (d+ > 3/4 of its slots) run one table pass per slice (support.cu) — in BOTH block
geometries, on graphs with closed-form answers (no config or fixture has such an owner: C5's
largest d+ is below it). K_n: every edge lies in n - 2 triangles, trussness n, one sub-level
(test_truss_serial.cpp's clique closed form at hub scale). Cocktail-party graph K_n minus a
perfect matching: every edge lies in n - 4 triangles and the graph is edge-transitive, so every
edge has trussness n - 2. Each case runs in its own process: the geometry override
(TDG_SUP_BIG) is read once per process."""
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def _clique_csr(n):
    ids = np.arange(n, dtype=np.int32)
    nb = np.broadcast_to(ids, (n, n))[~np.eye(n, dtype=bool)].reshape(n, n - 1)
    off = np.arange(n + 1, dtype=np.int64) * (n - 1)
    return n, n * (n - 1) // 2, off, np.ascontiguousarray(nb.reshape(-1))


def _cocktail_csr(n):
    assert n % 2 == 0
    ids = np.arange(n, dtype=np.int32)
    keep = ~np.eye(n, dtype=bool)
    keep[ids, ids ^ 1] = False  # drop the matching {2k, 2k+1}
    nb = np.broadcast_to(ids, (n, n))[keep].reshape(n, n - 2)
    off = np.arange(n + 1, dtype=np.int64) * (n - 2)
    return n, n * (n - 2) // 2, off, np.ascontiguousarray(nb.reshape(-1))


def run_case(kind: str, n: int) -> None:
    sys.path.insert(0, ROOT)
    from paper_1707_02000_b200 import trussdec
    n, m, off, nb = _clique_csr(n) if kind == "clique" else _cocktail_csr(n)
    tri_per_edge = n - 2 if kind == "clique" else n - 4
    ctx = trussdec.Context(0)
    g = trussdec.CsrGraph(n, m, off, nb)
    s, _ = ctx.support(g)
    assert s.min() == s.max() == tri_per_edge
    assert ctx.counters()["sup_hub"] > 0, "the sliced hub passes did not run"
    assert ctx.triangle_count(g) == m * tri_per_edge // 3
    truss, nsl, _, _ = ctx.truss(g)
    assert truss.min() == truss.max() == tri_per_edge + 2
    assert sum(nsl) == 1 and nsl[tri_per_edge] == 1  # the whole graph peels in one sub-level
    # the shards of the hub passes still sum to the supports
    parts = [ctx.support_shard(g, r, 3)[0].astype(np.uint64) for r in range(3)]
    assert np.array_equal(np.sum(parts, axis=0), s.astype(np.uint64))
    ctx.close()
    print("hub case ok", kind, n)


# (geometry, n): the small geometry's tables hold 3072 keys, the big one's 6144; a clique's owner
# lists make the device choose the big geometry, so the small one is forced for its case.
CASES = [("small", "clique", 3300), ("small", "cocktail", 3300), ("big", "clique", 6200)]


@pytest.mark.gpu
@pytest.mark.parametrize("geometry,kind,n", CASES)
def test_hub_slices_closed_form(geometry, kind, n):
    env = dict(os.environ)
    env.pop("TDG_SUP_BIG", None)
    if geometry == "small":
        env["TDG_SUP_BIG"] = "0"
    r = subprocess.run([sys.executable, os.path.abspath(__file__), kind, str(n)], capture_output=True, text=True,
                       timeout=900, env=env, cwd=ROOT)
    assert r.returncode == 0, (r.stdout + r.stderr)[-3000:]
    assert "hub case ok" in r.stdout


if __name__ == "__main__":
    run_case(sys.argv[1], int(sys.argv[2]))
