# U=3 default + support per-step own-edge aggregation (parity first); U=4 check
timeout 300 python -m pytest tests -m gpu -x -q -k "not config5" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
VARIANTS="base:;u4:-DTDG_PEEL_U=4" bash scripts/gpu_sweep11.sh
