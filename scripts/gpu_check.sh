set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc; free -g | head -2
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
tail -5 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q -k "not config5" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --config 1 --steps 3 --warmup 3 --no-e2e > gpurun_out/bench_c1.log 2>&1; echo "bench1 rc=$?"
tail -3 gpurun_out/bench_c1.log
timeout 600 python bench.py --config 3 --steps 2 --warmup 1 > gpurun_out/bench_c3.log 2>&1; echo "bench3 rc=$?"
tail -3 gpurun_out/bench_c3.log
