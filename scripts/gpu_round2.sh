# verify + measure after a change: GPU parity, C5 + C3 bench, C5 DRAM traffic (kernel replay),
# full ncu capture of k_peel and k_support at C3.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "not config5" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps ${STEPS:-3} --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; grep '^{' gpurun_out/bench.log | python scripts/summ.py
timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1; echo "bench c3 rc=$?"; grep '^{' gpurun_out/bench_c3.log | python scripts/summ.py
if [ -z "$NO_NCU" ]; then
timeout 900 ncu --replay-mode kernel --clock-control none --kernel-name-base function -k regex:'^k_(peel|support)$' \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
  --csv --log-file gpurun_out/traffic_c5.csv python scripts/run_one.py 5 > gpurun_out/ncu_traffic5.log 2>&1; echo "traffic5 rc=$?"; grep -v "^==" gpurun_out/traffic_c5.csv | tail -8
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:'^k_(peel|support)$' -c 2 \
  -o gpurun_out/full_c3 python scripts/run_one.py 3 > gpurun_out/ncu_full3.log 2>&1; echo "full3 rc=$?"; tail -3 gpurun_out/ncu_full3.log
fi
