# Re-entry check of HEAD: smoke, queued vs fused peel A/B at C3/C5, GPU parity, default bench.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv; nproc
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
V=paper_1707_02000_b200/lib_variants
for c in 3 5; do timeout 600 python scripts/run_one.py $c 2 > gpurun_out/ab_base_c$c.log 2>&1; echo "ab base c$c rc=$?"; tail -1 gpurun_out/ab_base_c$c.log; done
for c in 3 5; do TDG_SO=$V/fused/libtdg.so timeout 600 python scripts/run_one.py $c 2 > gpurun_out/ab_fused_c$c.log 2>&1; echo "ab fused c$c rc=$?"; tail -1 gpurun_out/ab_fused_c$c.log; done
timeout 300 python scripts/run_one.py 1 3 > gpurun_out/ab_base_c1.log 2>&1; tail -1 gpurun_out/ab_base_c1.log
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
timeout 1200 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; grep '^{' gpurun_out/bench.log | python scripts/summ.py
