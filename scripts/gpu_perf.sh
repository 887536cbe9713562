# perf exploration run: parity tests + benches on several configs
timeout 600 python -m pytest tests -m gpu -x -q -k "not config5" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for c in ${CONFIGS:-1 3 4}; do
  timeout 900 python bench.py --config $c --steps ${STEPS:-2} --warmup ${WARMUP:-1} --no-cpu-baseline > gpurun_out/bench_c$c.log 2>&1; echo "bench c$c rc=$?"
  python -c "
import json,sys
l=[x for x in open('gpurun_out/bench_c$c.log') if x.startswith('{')]
if not l: print(open('gpurun_out/bench_c$c.log').read()[-2000:]); sys.exit()
d=json.loads(l[-1]); print('C$c', 'value', round(d['value'],2), 'ms', round(d['ms_per_step'],1), {k:round(v,1) for k,v in d['phases_ms'].items()}, 'cfg', {k:d['config'][k] for k in ('m','sublevels','scans')}, 'e2e', d['e2e'] and round(d['e2e']['value'],2))
"
done
