# pieces rounded to whole 32*U-item steps (parity first)
timeout 300 python -m pytest tests -m gpu -x -q -k "not config5" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
VARIANTS="round:;noround:-DTDG_PIECE_ROUND=0" bash scripts/gpu_sweep11.sh
