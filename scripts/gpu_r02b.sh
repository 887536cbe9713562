# Bucketed global tables + bucketed support tables: parity, A/B variants, memcheck.
mkdir -p gpurun_out
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
V=paper_1707_02000_b200/lib_variants
for c in 3 5; do timeout 600 python scripts/run_one.py $c 2 > gpurun_out/ab_base_c$c.log 2>&1; echo "ab base c$c rc=$?"; tail -1 gpurun_out/ab_base_c$c.log; done
for v in hf3 fastbar supload4 suptab8k supu4; do for c in 3 5; do TDG_SO=$V/$v/libtdg.so timeout 600 python scripts/run_one.py $c 2 > gpurun_out/ab_${v}_c$c.log 2>&1; echo "ab $v c$c rc=$?"; tail -1 gpurun_out/ab_${v}_c$c.log; done; done
for v in base fastbar; do L=paper_1707_02000_b200/lib/libtdg.so; [ $v != base ] && L=$V/$v/libtdg.so; TDG_SO=$L timeout 300 python scripts/run_one.py 1 5 > gpurun_out/ab_${v}_c1.log 2>&1; echo "ab $v c1"; tail -2 gpurun_out/ab_${v}_c1.log; done
timeout 1800 compute-sanitizer --tool memcheck --error-exitcode 99 python scripts/sanitize.py > gpurun_out/memcheck.log 2>&1; echo "memcheck rc=$?"; tail -5 gpurun_out/memcheck.log
