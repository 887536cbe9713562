# Support pass rewrite (16-byte quads, shared-memory hit counters, hub passes): parity + variants.
mkdir -p gpurun_out
V=paper_1707_02000_b200/lib_variants
timeout 900 python -m pytest tests/test_truss_gpu.py tests/test_configs_gpu.py -m gpu -x -q > gpurun_out/pytest_sup.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_sup.log
for c in 3 5; do timeout 600 python scripts/run_one.py $c 2 > gpurun_out/sup_base_c$c.log 2>&1; echo "base c$c rc=$?"; tail -1 gpurun_out/sup_base_c$c.log; done
for v in u1b5 u1b4 u2b4 u2b3; do for c in 3 5; do TDG_SO=$V/$v/libtdg.so timeout 600 python scripts/run_one.py $c 2 > gpurun_out/sup_${v}_c$c.log 2>&1; echo "$v c$c rc=$?"; tail -1 gpurun_out/sup_${v}_c$c.log; done; done
