# DRAM bytes / L2 hit rate / L2 atomic + reduction sectors per launch of the hot kernels
# (ncu kernel replay) for the configs given as arguments; writes gpurun_out/ncu_traffic_C<c>.csv
# and the CUDA-source hash the capture belongs to (bench.py ties profiles/ncu_traffic.json to it).
# Usage (on the GPU box): bash scripts/ncu_traffic.sh 3 4 5
mkdir -p gpurun_out
python -c "import bench; print(bench.src_sha())" > gpurun_out/ncu_src_sha.txt
for c in "$@"; do
  timeout 900 python scripts/run_one.py $c > gpurun_out/plain_c$c.log 2>&1 &&
  timeout 1500 ncu --replay-mode kernel --clock-control none --kernel-name-base function \
    -k regex:'^k_(peel|support_tab)(<|$)' \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum,lts__t_requests_op_atom.sum,lts__t_requests_op_red.sum,sm__inst_executed.sum \
    --csv --log-file gpurun_out/ncu_traffic_C$c.csv python scripts/run_one.py $c > gpurun_out/ncu_traffic_C$c.log 2>&1
  echo "ncu traffic C$c rc=$?"
done
