# Round-end evidence on the final code: smoke, full GPU parity (incl. C5 golden), default
# bench (C5), C1-C4 benches, ncu launch list, C5 DRAM traffic, full capture at C3.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv; nproc
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; grep '^{' gpurun_out/bench.log | python scripts/summ.py
for c in 1 2 3 4; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c$c.log 2>&1; echo "bench c$c rc=$?"; grep '^{' gpurun_out/bench_c$c.log | python scripts/summ.py; done
if [ -z "$NO_NCU" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c5.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --replay-mode kernel --clock-control none --kernel-name-base function -k regex:'^k_(peel|support_tab)$' \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
  --csv --log-file gpurun_out/traffic_c5.csv python scripts/run_one.py 5 > gpurun_out/ncu_traffic5.log 2>&1; echo "traffic5 rc=$?"; grep -v "^==" gpurun_out/traffic_c5.csv | tail -8
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:'^k_(peel|support_tab)$' -c 2 \
  -o gpurun_out/full_c3 python scripts/run_one.py 3 > gpurun_out/ncu_full3.log 2>&1; echo "full3 rc=$?"; tail -2 gpurun_out/ncu_full3.log
fi
