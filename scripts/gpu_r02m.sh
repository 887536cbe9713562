mkdir -p gpurun_out
V=paper_1707_02000_b200/lib_variants
for v in ncrb0 ncrb13 ncrb12 st0; do for c in 3 5; do TDG_SO=$V/$v/libtdg.so timeout 600 python scripts/run_one.py $c 2 > gpurun_out/m_${v}_c$c.log 2>&1; echo "$v c$c rc=$?"; tail -1 gpurun_out/m_${v}_c$c.log | cut -c1-100; tail -1 gpurun_out/m_${v}_c$c.log | grep -o "'support_ms.*process_ms[^,]*\|'rebuild_ms.*"; done; done
