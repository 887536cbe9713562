# support multiplicative table hash (parity first), filter density 16 / 8 / 4 bits per key
timeout 300 python -m pytest tests -m gpu -x -q -k "not config5" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
VARIANTS="base:;fs2:-DTDG_FSHIFT=2;fs3:-DTDG_FSHIFT=3" CONFIGS="3 5" bash scripts/gpu_sweep5.sh
