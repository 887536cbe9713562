# Arena trims + guided pieces + fast barrier + checked build: parity, A/B, bench, ncu.
mkdir -p gpurun_out
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 2000 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
V=paper_1707_02000_b200/lib_variants
for c in 3 5; do timeout 600 python scripts/run_one.py $c 2 > gpurun_out/ab_base_c$c.log 2>&1; echo "ab base c$c rc=$?"; tail -1 gpurun_out/ab_base_c$c.log; done
for v in hf3 noguided gridsync; do for c in 3 5; do TDG_SO=$V/$v/libtdg.so timeout 600 python scripts/run_one.py $c 2 > gpurun_out/ab_${v}_c$c.log 2>&1; echo "ab $v c$c rc=$?"; tail -1 gpurun_out/ab_${v}_c$c.log; done; done
timeout 300 python scripts/run_one.py 1 3 > gpurun_out/ab_base_c1.log 2>&1; tail -1 gpurun_out/ab_base_c1.log
timeout 1500 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; grep '^{' gpurun_out/bench.log | python scripts/summ.py
if [ -z "$NO_NCU" ]; then
bash scripts/ncu_traffic.sh 3 5
timeout 300 python scripts/run_one.py 3 > gpurun_out/plain3.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:'^k_support_tab' -c 1 \
  -o gpurun_out/full_c3_sup python scripts/run_one.py 3 > gpurun_out/ncu_full3_sup.log 2>&1; echo "full3 sup rc=$?"
timeout 300 python scripts/run_one.py 3 > gpurun_out/plain3.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:'^k_peel(<|$)' -c 1 \
  -o gpurun_out/full_c3_peel python scripts/run_one.py 3 > gpurun_out/ncu_full3_peel.log 2>&1; echo "full3 peel rc=$?"
fi
