# A/B of lib_variants (scripts/variants.sh) on the configs in $CFGS (default "5 3"): peel / support / total per variant.
mkdir -p gpurun_out
for c in ${CFGS:-5 3}; do
  for v in base $VARS; do
    so=paper_1707_02000_b200/lib_variants/$v/libtdg.so; [ $v = base ] && so=paper_1707_02000_b200/lib/libtdg.so
    TDG_SO=$so timeout 900 python scripts/run_one.py $c ${REPS:-3} > gpurun_out/ab_${v}_c$c.log 2>&1
    echo "$v c$c: $(tail -1 gpurun_out/ab_${v}_c$c.log | grep -o "parity=[a-zA-Z]*") $(tail -1 gpurun_out/ab_${v}_c$c.log | grep -o "'build_ms.*")"
  done
done
