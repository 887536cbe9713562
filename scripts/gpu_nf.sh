# near/far scan + membership filters: parity, then C3/C5 timings (short timeouts: a hung
# cooperative kernel must not eat the budget)
summ() { python -c "
import sys,ast
for l in sys.stdin:
    if not l.startswith('C') or '{' not in l: continue
    d=ast.literal_eval(l[l.index('{'):])
    print({k:d.get(k) for k in ('support_ms','peel_ms','scan_ms','process_ms','compact_ms','total_ms','scans','compactions')})"; }
timeout 300 python -m pytest tests -m gpu -x -q -k "not config5" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for f in 1 0; do for c in ${CONFIGS:-3 5}; do echo "== filter=$f C$c"; TDG_PEEL_FILTER=$f timeout 240 python scripts/run_one.py $c 2 2>&1 | summ; done; done
IFS=';' read -ra VS <<< "${VARIANTS:-nf16d2:-DTDG_NEAR_ADD=16 -DTDG_NEAR_DIV=2;off:-DTDG_NEAR_ADD=2000000000 -DTDG_NEAR_DIV=1;fmin256:-DTDG_FMIN=256;fmin4k:-DTDG_FMIN=4096}"
for v in "${VS[@]}"; do
  name="${v%%:*}"; flags="${v#*:}"
  touch paper_1707_02000_b200/csrc/peel.cu paper_1707_02000_b200/csrc/build.cu; make -s -C paper_1707_02000_b200/csrc -j16 NVEXTRA="$flags" 2>&1 | grep -E "error"
  for c in ${CONFIGS:-3 5}; do echo "== $name C$c"; timeout 240 python scripts/run_one.py $c 2 2>&1 | summ; done
done
touch paper_1707_02000_b200/csrc/peel.cu paper_1707_02000_b200/csrc/build.cu; make -s -C paper_1707_02000_b200/csrc -j16 2>&1 | grep error
