# One verification + measurement round on the GPU box: smoke, GPU parity, default bench (C5),
# ncu launch list of a 1-step bench, DRAM traffic of the top kernels (application replay).
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv; nproc
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q -k "not config5" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -c 3000 gpurun_out/bench.log
if [ -z "$NO_NCU" ]; then
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c5.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "launches rc=$?"
CFG=5 timeout 900 bash scripts/gpu_traffic.sh
fi
