mkdir -p gpurun_out
run() { echo "$1 $(tail -1 gpurun_out/q.log | grep -o "parity=[a-zA-Z]*") $(tail -1 gpurun_out/q.log | grep -o "peel_ms[^,]*") $(tail -1 gpurun_out/q.log | grep -o "rebuild_ms.*")"; }
for r in 1/4/3 1/3/5 1/4/5 2/5/6 1/2/6 1/6/3; do for c in 3 5; do TDG_REBUILD=$r timeout 600 python scripts/run_one.py $c 2 > gpurun_out/q.log 2>&1; run "rb=$r c$c"; done; done
for c in 3 5; do TDG_PEEL_FILTER=0 timeout 600 python scripts/run_one.py $c 2 > gpurun_out/q.log 2>&1; run "nofilter c$c"; done
for v in fmin64 fmin32; do for c in 3 5; do TDG_SO=paper_1707_02000_b200/lib_variants/$v/libtdg.so timeout 600 python scripts/run_one.py $c 2 > gpurun_out/q.log 2>&1; run "$v c$c"; done; done
