# own-slot state read placement (TDG_PEEL_EA 0/1/2), U=3; hit / dead-probe counters once
summ() { python -c "
import sys,ast
for l in sys.stdin:
    if not l.startswith('C') or '{' not in l: continue
    d=ast.literal_eval(l[l.index('{'):])
    print({k:d.get(k) for k in ('support_ms','peel_ms','scan_ms','process_ms','compact_ms','total_ms','probes','hits','dead_probes')})"; }
timeout 900 python -m pytest tests -m gpu -x -q -k "not config5" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
for c in 3 5; do echo "== counters C$c"; TDG_COUNT_HITS=1 timeout 600 python scripts/run_one.py $c 1 2>&1 | summ; done
IFS=';' read -ra VS <<< "${VARIANTS:-ea1:;ea0:-DTDG_PEEL_EA=0;ea2:-DTDG_PEEL_EA=2}"
for v in "${VS[@]}"; do
  name="${v%%:*}"; flags="${v#*:}"
  touch paper_1707_02000_b200/csrc/peel.cu; make -s -C paper_1707_02000_b200/csrc -j16 NVEXTRA="$flags" 2>&1 | grep -E "error"
  for c in ${CONFIGS:-3 5}; do echo "== $name C$c"; timeout 600 python scripts/run_one.py $c 2 2>&1 | summ; done
done
touch paper_1707_02000_b200/csrc/peel.cu; make -s -C paper_1707_02000_b200/csrc -j16 2>&1 | grep error
