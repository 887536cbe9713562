# engine pieces per warp; current per-sub-level trace at C5
VARIANTS="p8:-DTDG_PIECES=8ull;p2:-DTDG_PIECES=2ull" bash scripts/gpu_sweep11.sh
TDG_TRACE=gpurun_out/trace_c5.txt timeout 240 python scripts/run_one.py 5 1 > /dev/null 2>&1; echo "trace rc=$?"
