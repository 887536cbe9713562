# Round-2 checkpoint: smoke, GPU parity, bench (C5 + C4 same-config pair + byte model), C1/C3
# benches, sub-level traces, ncu traffic (C3, C5) and full captures of the two hot kernels (C3).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv; nproc
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
V=paper_1707_02000_b200/lib_variants
TDG_SO=$V/mergeall/libtdg.so timeout 900 python -m pytest tests/test_truss_gpu.py tests/test_configs_gpu.py -x -q -k "not config5" > gpurun_out/pytest_mergeall.log 2>&1; echo "pytest mergeall rc=$?"; tail -3 gpurun_out/pytest_mergeall.log
for v in nomerge merge8 mmin64 hf3; do for c in 3 5; do TDG_SO=$V/$v/libtdg.so timeout 600 python scripts/run_one.py $c 2 > gpurun_out/ab_${v}_c$c.log 2>&1; echo "ab $v c$c rc=$?"; tail -1 gpurun_out/ab_${v}_c$c.log; done; done
for c in 3 5; do timeout 600 python scripts/run_one.py $c 2 > gpurun_out/ab_base_c$c.log 2>&1; echo "ab base c$c rc=$?"; tail -1 gpurun_out/ab_base_c$c.log; done
timeout 1500 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; grep '^{' gpurun_out/bench.log | python scripts/summ.py
for c in 1 3; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c$c.log 2>&1; echo "bench c$c rc=$?"; grep '^{' gpurun_out/bench_c$c.log | python scripts/summ.py; done
TDG_TRACE=gpurun_out/trace_c1.txt timeout 300 python scripts/run_one.py 1 2 > gpurun_out/trace_c1.log 2>&1; echo "trace c1 rc=$?"
TDG_TRACE=gpurun_out/trace_c5.txt timeout 600 python scripts/run_one.py 5 1 > gpurun_out/trace_c5.log 2>&1; echo "trace c5 rc=$?"
if [ -z "$NO_NCU" ]; then
bash scripts/ncu_traffic.sh 3 5
timeout 300 python scripts/run_one.py 3 > gpurun_out/plain3.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:'^k_support_tab' -c 1 \
  -o gpurun_out/full_c3_sup python scripts/run_one.py 3 > gpurun_out/ncu_full3_sup.log 2>&1; echo "full3 sup rc=$?"; tail -2 gpurun_out/ncu_full3_sup.log
timeout 300 python scripts/run_one.py 3 > gpurun_out/plain3.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:'^k_peel(<|$)' -c 1 \
  -o gpurun_out/full_c3_peel python scripts/run_one.py 3 > gpurun_out/ncu_full3_peel.log 2>&1; echo "full3 peel rc=$?"; tail -2 gpurun_out/ncu_full3_peel.log
fi
