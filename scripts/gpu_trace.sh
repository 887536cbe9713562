# Per-sub-level traces (TDG_TRACE) of C1 / C3 / C5 summarised by size class, plus the shard tests.
mkdir -p gpurun_out
for c in ${CFGS:-1 3 5}; do
  TDG_TRACE=gpurun_out/trace_c$c.txt timeout 600 python scripts/run_one.py $c 1 > gpurun_out/trace_run_c$c.log 2>&1; tail -1 gpurun_out/trace_run_c$c.log
  python scripts/trace_classes.py gpurun_out/trace_c$c.txt > gpurun_out/trace_classes_c$c.md; cat gpurun_out/trace_classes_c$c.md
  [ $c = 5 ] && rm -f gpurun_out/trace_c5.txt
done
timeout 600 python -m pytest tests/test_support_shard_gpu.py -x -q 2>&1 | tail -3
