# Per-launch DRAM traffic + L1/L2 sector mix of k_peel / k_support (application replay) on config $CFG
CFG=${CFG:-3}
CMD="python scripts/run_one.py $CFG"
mkdir -p gpurun_out
$CMD > gpurun_out/mix_plain_c$CFG.log 2>&1 && echo "plain ok" &&
ncu --replay-mode application --clock-control none --kernel-name-base function -k regex:'^k_(peel|support)$' \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_atom.sum,lts__t_sectors_srcunit_tex_op_red.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,lts__t_sectors_srcunit_tex_op_atom_lookup_miss.sum,lts__t_sectors_srcunit_tex_op_red_lookup_miss.sum,dram__sectors_read.sum,dram__sectors_write.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_hit.sum,smsp__inst_executed.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed \
  --csv --log-file gpurun_out/mix_c$CFG.csv $CMD > gpurun_out/ncu_mix_c$CFG.log 2>&1; echo "ncu rc=$?"
