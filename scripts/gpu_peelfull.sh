# full ncu section set for the cooperative k_peel via application replay (kernel replay returns n/a)
timeout 1500 ncu --set full --replay-mode application --clock-control none --kernel-name-base function -k regex:'^k_peel$' -c 1 \
  -o gpurun_out/peel_full_c3 python scripts/run_one.py 3 > gpurun_out/ncu_peelfull.log 2>&1; echo "rc=$?"; tail -3 gpurun_out/ncu_peelfull.log
