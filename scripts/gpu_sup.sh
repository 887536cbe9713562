# support pass forms: parity first, then A/B timings (owner-table vs global search, table sizes)
summ() { python -c "
import sys,ast
for l in sys.stdin:
    if not l.startswith('C') or '{' not in l: continue
    d=ast.literal_eval(l[l.index('{'):])
    print({k:d.get(k) for k in ('support_ms','peel_ms','total_ms','support_probes','triangles')})"; }
timeout 900 python -m pytest tests -m gpu -x -q -k "not config5" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for c in ${CONFIGS:-3 5}; do
  for f in tab search; do echo "== $f C$c"; TDG_SUP_FORM=$f timeout 600 python scripts/run_one.py $c 2 2>&1 | summ; done
done
touch paper_1707_02000_b200/csrc/support.cu; make -s -C paper_1707_02000_b200/csrc -j16 NVEXTRA=-DTDG_SUP_TAB=8192 2>&1 | grep error
for c in ${CONFIGS:-3 5}; do echo "== tab8192 C$c"; timeout 600 python scripts/run_one.py $c 2 2>&1 | summ; done
touch paper_1707_02000_b200/csrc/support.cu; make -s -C paper_1707_02000_b200/csrc -j16 2>&1 | grep error
