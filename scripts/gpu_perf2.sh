# perf + counters: one decomposition per config with hit counting (diagnostic), then plain benches
for c in ${CONFIGS:-3}; do TDG_COUNT_HITS=1 timeout 900 python scripts/run_one.py $c 1 2>&1 | tail -1; done
