CMD="python scripts/run_one.py ${CFG:-3}"
$CMD > gpurun_out/prof2_plain.log 2>&1 && echo "plain ok" && tail -1 gpurun_out/prof2_plain.log &&
ncu --replay-mode application --clock-control none --import-source on --kernel-name-base function -k regex:'^k_peel$' -c 1 \
  --section SpeedOfLight --section MemoryWorkloadAnalysis --section WarpStateStats --section SourceCounters --section LaunchStats --section Occupancy --section ComputeWorkloadAnalysis \
  -o gpurun_out/prof_peel_c${CFG:-3} $CMD > gpurun_out/ncu_peel.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_peel.log
