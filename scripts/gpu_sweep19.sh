# hash-table slot loads through the read-only path
VARIANTS="nc:-DTDG_HTAB_NC=1;base:" bash scripts/gpu_sweep11.sh
