# L2 persisting window for the processed bitmap + register/occupancy variants; checked
# build; C1-C4 benches; C5 launch list.
mkdir -p gpurun_out
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 2000 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
V=paper_1707_02000_b200/lib_variants
for c in 3 5; do timeout 600 python scripts/run_one.py $c 2 > gpurun_out/ab_base_c$c.log 2>&1; echo "ab base c$c rc=$?"; tail -1 gpurun_out/ab_base_c$c.log; done
for v in nopersist m3 u4m3 u2 hf3; do for c in 3 5; do TDG_SO=$V/$v/libtdg.so timeout 600 python scripts/run_one.py $c 2 > gpurun_out/ab_${v}_c$c.log 2>&1; echo "ab $v c$c rc=$?"; tail -1 gpurun_out/ab_${v}_c$c.log; done; done
for c in 1 2 3 4; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c$c.log 2>&1; echo "bench c$c rc=$?"; grep '^{' gpurun_out/bench_c$c.log | python scripts/summ.py; done
timeout 900 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-counts > gpurun_out/plain_launch.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c5.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-counts > gpurun_out/ncu_launch.log 2>&1; echo "launches rc=$?"
