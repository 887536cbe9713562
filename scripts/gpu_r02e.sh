# Two-stage (queued) peel probes: parity + A/B vs the fused chain.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,clocks.max.mem,power.draw,temperature.gpu,utilization.gpu --format=csv
nvidia-smi --query-compute-apps=pid,used_memory --format=csv
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 2000 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
V=paper_1707_02000_b200/lib_variants
for round in 1 2; do
for c in 3 5; do timeout 600 python scripts/run_one.py $c 2 > gpurun_out/ab_base_c$c.log 2>&1; echo "ab base c$c rc=$?"; tail -1 gpurun_out/ab_base_c$c.log; done
for v in fused hf3; do for c in 3 5; do TDG_SO=$V/$v/libtdg.so timeout 600 python scripts/run_one.py $c 2 > gpurun_out/ab_${v}_c$c.log 2>&1; echo "ab $v c$c rc=$?"; tail -1 gpurun_out/ab_${v}_c$c.log; done; done
done
timeout 300 python scripts/run_one.py 1 3 > gpurun_out/ab_base_c1.log 2>&1; tail -1 gpurun_out/ab_base_c1.log
