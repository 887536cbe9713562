# peel engine fast path and pieces per warp on the final build
VARIANTS="fast:-DTDG_PEEL_FAST=1;p8:-DTDG_PIECES=8ull;p6:-DTDG_PIECES=6ull" bash scripts/gpu_sweep11.sh
