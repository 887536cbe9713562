CMD="python scripts/run_one.py ${CFG:-5}"
$CMD > gpurun_out/profsup_plain.log 2>&1 && echo "plain ok" && tail -1 gpurun_out/profsup_plain.log | cut -c1-200 &&
ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:'^k_support$' -c 1 -o gpurun_out/prof_support_c${CFG:-5} $CMD > gpurun_out/ncu_sup.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/ncu_sup.log
