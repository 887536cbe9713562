mkdir -p gpurun_out
run() { echo "$1 $(tail -1 gpurun_out/q.log | grep -o "parity=[a-zA-Z]*") $(tail -1 gpurun_out/q.log | grep -o "peel_ms[^,]*") $(tail -1 gpurun_out/q.log | grep -o "rebuild_ms.*")"; }
for v in $VARS; do for r in 1/4/3 1/2/4; do for c in 1 3 5; do TDG_SO=paper_1707_02000_b200/$v/libtdg.so TDG_REBUILD=$r timeout 600 python scripts/run_one.py $c 2 > gpurun_out/q.log 2>&1; run "$v rb=$r c$c"; done; done; done
