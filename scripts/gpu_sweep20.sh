# minimum engine piece size x pieces per warp
VARIANTS="ps384:-DTDG_MIN_PIECE=384ull;ps384p8:-DTDG_MIN_PIECE=384ull -DTDG_PIECES=8ull;ps1k8:-DTDG_MIN_PIECE=1024ull -DTDG_PIECES=8ull" bash scripts/gpu_sweep11.sh
