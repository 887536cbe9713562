# peel knobs re-checked on the U=2 / no-staging build
VARIANTS="base:;m5:-DTDG_PEEL_MINB=5;s256k:-DTDG_SORT_MIN=262144;s4m:-DTDG_SORT_MIN=4194304;c85:-DTDG_COMPACT_NUM=85 -DTDG_COMPACT_DEN=100" CONFIGS="3 5" bash scripts/gpu_sweep5.sh
