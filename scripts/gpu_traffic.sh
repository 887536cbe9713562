# DRAM traffic per launch of the top kernels (application replay, few metrics) for bench's roofline.traffic
CMD="python scripts/run_one.py ${CFG:-5}"
$CMD > gpurun_out/traffic_plain.log 2>&1 && echo "plain ok" &&
ncu --replay-mode application --clock-control none --kernel-name-base function -k regex:'^k_(peel|support)$' \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active \
  --csv --log-file gpurun_out/traffic_c${CFG:-5}.csv $CMD > gpurun_out/ncu_traffic.log 2>&1; echo "ncu rc=$?"; cat gpurun_out/traffic_c${CFG:-5}.csv | tail -14
