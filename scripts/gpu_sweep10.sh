# filter density / bits per key around the new default (4 bits/key), small-table smem build; parity first
timeout 300 python -m pytest tests -m gpu -x -q -k "not config5" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
VARIANTS="base:;fs4:-DTDG_FSHIFT=4;fs3k2:-DTDG_FK=2;fs4k2:-DTDG_FSHIFT=4 -DTDG_FK=2;fs3min256:-DTDG_FMIN=256" CONFIGS="3 5" bash scripts/gpu_sweep5.sh
