# support pass: probe items per lane per step (TDG_SUP_U 2 default vs 1); parity first
summ() { python -c "
import sys,ast
for l in sys.stdin:
    if not l.startswith('C') or '{' not in l: continue
    d=ast.literal_eval(l[l.index('{'):])
    print({k:d.get(k) for k in ('build_ms','support_ms','peel_ms','process_ms','total_ms')})"; }
timeout 300 python -m pytest tests -m gpu -x -q -k "not config5" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
for c in 3 5; do echo "== supU2 C$c"; timeout 240 python scripts/run_one.py $c 2 2>&1 | summ; done
touch paper_1707_02000_b200/csrc/support.cu; make -s -C paper_1707_02000_b200/csrc -j16 NVEXTRA=-DTDG_SUP_U=1 2>&1 | grep error
for c in 3 5; do echo "== supU1 C$c"; timeout 240 python scripts/run_one.py $c 2 2>&1 | summ; done
touch paper_1707_02000_b200/csrc/support.cu; make -s -C paper_1707_02000_b200/csrc -j16 NVEXTRA=-DTDG_SUP_U=4 2>&1 | grep error
for c in 3 5; do echo "== supU4 C$c"; timeout 240 python scripts/run_one.py $c 2 2>&1 | summ; done
touch paper_1707_02000_b200/csrc/support.cu; make -s -C paper_1707_02000_b200/csrc -j16 2>&1 | grep error
