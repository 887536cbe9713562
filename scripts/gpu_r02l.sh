# In-peel table rebuild on the live graph: parity + A/B of the rebuild threshold.
mkdir -p gpurun_out
V=paper_1707_02000_b200/lib_variants
timeout 900 python -m pytest tests/test_truss_gpu.py tests/test_configs_gpu.py tests/test_checked_gpu.py -m gpu -x -q > gpurun_out/pytest_l.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_l.log
for c in 1 3 4 5; do timeout 600 python scripts/run_one.py $c 2 > gpurun_out/l_base_c$c.log 2>&1; echo "base c$c rc=$?"; tail -1 gpurun_out/l_base_c$c.log | cut -c1-420; done
for v in rb0 rb23 rb13 rb34; do for c in 3 5; do TDG_SO=$V/$v/libtdg.so timeout 600 python scripts/run_one.py $c 2 > gpurun_out/l_${v}_c$c.log 2>&1; echo "$v c$c rc=$?"; tail -1 gpurun_out/l_${v}_c$c.log | cut -c1-420; done; done
TDG_TRACE=gpurun_out/l_trace_c5.txt timeout 600 python scripts/run_one.py 5 1 > gpurun_out/l_trace_c5.log 2>&1; python scripts/trace_classes.py gpurun_out/l_trace_c5.txt
