# Static-tier / fused-prep A/B (the head regressed the C5 peel 2.37 -> 2.66 s), C5 task-shape histogram, C5 trace.
mkdir -p gpurun_out
V=paper_1707_02000_b200/lib_variants
for c in 1 3 5; do timeout 600 python scripts/run_one.py $c 2 > gpurun_out/k_base_c$c.log 2>&1; echo "base c$c rc=$?"; tail -1 gpurun_out/k_base_c$c.log | cut -c1-400; done
for v in st2 st0 nofuse; do for c in 1 3 5; do TDG_SO=$V/$v/libtdg.so timeout 600 python scripts/run_one.py $c 2 > gpurun_out/k_${v}_c$c.log 2>&1; echo "$v c$c rc=$?"; tail -1 gpurun_out/k_${v}_c$c.log | cut -c1-400; done; done
TDG_SO=$V/diag/libtdg.so timeout 600 python scripts/run_one.py 5 1 > gpurun_out/k_diag_c5.log 2>&1; grep DIAG gpurun_out/k_diag_c5.log
TDG_SO=$V/diag/libtdg.so timeout 600 python scripts/run_one.py 3 1 > gpurun_out/k_diag_c3.log 2>&1; grep DIAG gpurun_out/k_diag_c3.log
TDG_TRACE=gpurun_out/k_trace_c5.txt timeout 600 python scripts/run_one.py 5 1 > gpurun_out/k_trace_c5.log 2>&1; python scripts/trace_classes.py gpurun_out/k_trace_c5.txt
TDG_TRACE=gpurun_out/k_trace_c1.txt timeout 600 python scripts/run_one.py 1 2 > gpurun_out/k_trace_c1.log 2>&1; python scripts/trace_classes.py gpurun_out/k_trace_c1.txt
