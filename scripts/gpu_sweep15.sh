# peel U / block shape re-checked with task descriptors
VARIANTS="u3:-DTDG_PEEL_U=3;t512:-DTDG_PEEL_THREADS=512 -DTDG_PEEL_MINB=2;p8:-DTDG_PIECES=8ull" bash scripts/gpu_sweep11.sh
