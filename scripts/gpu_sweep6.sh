# U=2 follow-ups (staging off, 3 blocks/SM); parity first (support table / visit changes)
timeout 300 python -m pytest tests -m gpu -x -q -k "not config5" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
VARIANTS="u2:;u2nostage:-DTDG_STAGE_MIN=0;u2m3:-DTDG_PEEL_MINB=3" bash scripts/gpu_sweep5.sh
