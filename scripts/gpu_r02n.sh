mkdir -p gpurun_out
V=paper_1707_02000_b200/lib_variants
for v in $VARS; do for c in 3 5; do TDG_SO=$V/$v/libtdg.so timeout 600 python scripts/run_one.py $c 2 > gpurun_out/n_${v}_c$c.log 2>&1; echo "$v c$c rc=$? $(tail -1 gpurun_out/n_${v}_c$c.log | grep -o 'parity=[a-zA-Z]*') $(tail -1 gpurun_out/n_${v}_c$c.log | grep -o "'peel_ms[^,]*") $(tail -1 gpurun_out/n_${v}_c$c.log | grep -o "'rebuild_ms.*")"; done; done
