CMD="python scripts/run_one.py ${CFG:-3}"
$CMD > gpurun_out/l2mix_plain.log 2>&1 && echo "plain ok" &&
ncu --replay-mode application --clock-control none --kernel-name-base function -k regex:'^k_(peel|support)$' \
  --metrics lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_atom.sum,lts__t_sectors_srcunit_tex_op_red.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,lts__t_sectors_srcunit_tex_op_atom_lookup_miss.sum,lts__t_sectors_srcunit_tex_op_red_lookup_miss.sum,dram__sectors_read.sum,dram__sectors_write.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_hit.sum \
  --csv --log-file gpurun_out/l2mix_c${CFG:-3}.csv $CMD > gpurun_out/ncu_l2mix.log 2>&1; echo "ncu rc=$?"
