# ncu evidence: launch list of one bench step, then --set full on k_peel and k_support (C3)
CMD="python bench.py --config ${CFG:-3} --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/prof_plain.log 2>&1 && echo "plain ok" &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "launches rc=$?"
$CMD > gpurun_out/prof_plain2.log 2>&1 &&
ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:'^k_(peel|support)$' -c 2 -o gpurun_out/prof_c${CFG:-3} $CMD > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"
tail -5 gpurun_out/ncu_full.log
