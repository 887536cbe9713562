# No L2 persisting window: queued vs fused peel A/B at C3/C5 (2 rounds); C1; ncu full capture of
# k_support_tab and k_peel at C3 with source.
mkdir -p gpurun_out
V=paper_1707_02000_b200/lib_variants
for round in 1 2; do
for c in 3 5; do timeout 600 python scripts/run_one.py $c 2 > gpurun_out/ab_base_c$c.log 2>&1; echo "ab base c$c rc=$?"; tail -1 gpurun_out/ab_base_c$c.log; done
for c in 3 5; do TDG_SO=$V/fused/libtdg.so timeout 600 python scripts/run_one.py $c 2 > gpurun_out/ab_fused_c$c.log 2>&1; echo "ab fused c$c rc=$?"; tail -1 gpurun_out/ab_fused_c$c.log; done
done
timeout 300 python scripts/run_one.py 1 3 > gpurun_out/ab_base_c1.log 2>&1; tail -1 gpurun_out/ab_base_c1.log
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:'^k_support_tab$' -c 1 \
  -o gpurun_out/full_sup_c3 python scripts/run_one.py 3 > gpurun_out/ncu_full_sup3.log 2>&1; echo "fullsup rc=$?"; tail -2 gpurun_out/ncu_full_sup3.log
