# Rebuild as separate kernels between k_peel segments: parity + thresholds on one binary, U = 2 vs 3.
mkdir -p gpurun_out
V=paper_1707_02000_b200/lib_variants
timeout 900 python -m pytest tests/test_truss_gpu.py tests/test_configs_gpu.py tests/test_checked_gpu.py tests/test_shim_gpu.py -m gpu -x -q > gpurun_out/pytest_p.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_p.log
for so in lib/libtdg.so lib_variants/u2/libtdg.so; do for r in 0/0 1/2 1/4 1/8; do for c in 1 3 5; do TDG_SO=paper_1707_02000_b200/$so TDG_REBUILD=$r timeout 600 python scripts/run_one.py $c 2 > gpurun_out/p.log 2>&1; echo "$so rb=$r c$c rc=$? $(tail -1 gpurun_out/p.log | grep -o "parity=[a-zA-Z]*") $(tail -1 gpurun_out/p.log | grep -o "peel_ms[^,]*") $(tail -1 gpurun_out/p.log | grep -o "rebuild_ms.*")"; done; done; done
