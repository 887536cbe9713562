# parity + C3/C5 timing after an engine/build change
summ() { python -c "
import sys,ast
for l in sys.stdin:
    if not l.startswith('C') or '{' not in l: continue
    d=ast.literal_eval(l[l.index('{'):])
    print({k:d.get(k) for k in ('build_ms','support_ms','peel_ms','scan_ms','process_ms','compact_ms','total_ms')})"; }
timeout 400 python -m pytest tests -m gpu -x -q -k "not config5" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for c in ${CONFIGS:-3 5}; do echo "== C$c"; timeout 240 python scripts/run_one.py $c 2 2>&1 | summ; done
if [ -n "$TRACE" ]; then TDG_TRACE=gpurun_out/trace_c5.txt timeout 240 python scripts/run_one.py 5 1 > /dev/null 2>&1; echo "trace rc=$?"; fi
