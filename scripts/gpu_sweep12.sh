# support U / table density at 5 blocks/SM; peel bucket granularity (parity first)
timeout 300 python -m pytest tests -m gpu -x -q -k "not config5" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
VARIANTS="base:;supu3:-DTDG_SUP_U=3;load8:-DTDG_SUP_LOAD=8;bk18:-DTDG_BUCKET_BITS=18;bk20:-DTDG_BUCKET_BITS=20" bash scripts/gpu_sweep11.sh
