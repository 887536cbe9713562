# Re-entry check of head: full GPU parity, C1/C3/C5 phase times.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv; nproc
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for c in 1 3 4 5; do timeout 600 python scripts/run_one.py $c 3 > gpurun_out/head_c$c.log 2>&1; echo "c$c rc=$?"; tail -1 gpurun_out/head_c$c.log; done
