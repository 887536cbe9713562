# last knobs on the final build: compaction trigger, filter threshold
VARIANTS="c85:-DTDG_COMPACT_NUM=85 -DTDG_COMPACT_DEN=100;fmin512:-DTDG_FMIN=512;fmin2k:-DTDG_FMIN=2048" bash scripts/gpu_sweep11.sh
