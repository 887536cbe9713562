# peel block size 512 (fewer blocks per grid barrier); support table-segment threshold (parity first)
timeout 300 python -m pytest tests -m gpu -x -q -k "not config5" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
VARIANTS="t512:-DTDG_PEEL_THREADS=512 -DTDG_PEEL_MINB=2;seg256:-DTDG_SUP_SEGMIN=256u;segdiv2:-DTDG_SUP_SEGDIV=2u -DTDG_SUP_SEGMIN=512u;seg2k:-DTDG_SUP_SEGMIN=2048u" bash scripts/gpu_sweep11.sh
