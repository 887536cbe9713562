# Full ncu capture of k_support_tab at C3 (source-level), for scripts/sass_by_line.py.
mkdir -p gpurun_out
timeout 600 python scripts/run_one.py 3 1 > gpurun_out/plain_c3.log 2>&1 && tail -1 gpurun_out/plain_c3.log
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:'^k_support_tab$' -c 1 \
  -o gpurun_out/full_sup_c3 -f python scripts/run_one.py 3 > gpurun_out/ncu_full_sup.log 2>&1; echo "rc=$?"; tail -2 gpurun_out/ncu_full_sup.log
