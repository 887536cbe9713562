# peel knobs with filters + near/far: compaction trigger, bucket-sort threshold, staging
summ() { python -c "
import sys,ast
for l in sys.stdin:
    if not l.startswith('C') or '{' not in l: continue
    d=ast.literal_eval(l[l.index('{'):])
    print({k:d.get(k) for k in ('build_ms','support_ms','peel_ms','scan_ms','process_ms','compact_ms','total_ms')})"; }
IFS=';' read -ra VS <<< "${VARIANTS:-c80:-DTDG_COMPACT_NUM=8 -DTDG_COMPACT_DEN=10;c95:-DTDG_COMPACT_NUM=95 -DTDG_COMPACT_DEN=100;s256k:-DTDG_SORT_MIN=262144;s4m:-DTDG_SORT_MIN=4194304;nostage:-DTDG_STAGE_MIN=0;u2:-DTDG_PEEL_U=2}"
for v in "${VS[@]}"; do
  name="${v%%:*}"; flags="${v#*:}"
  touch paper_1707_02000_b200/csrc/peel.cu paper_1707_02000_b200/csrc/build.cu paper_1707_02000_b200/csrc/capi.cu; make -s -C paper_1707_02000_b200/csrc -j16 NVEXTRA="$flags" 2>&1 | grep -E "error"
  for c in ${CONFIGS:-3 5}; do echo "== $name C$c"; timeout 240 python scripts/run_one.py $c 2 2>&1 | summ; done
done
touch paper_1707_02000_b200/csrc/peel.cu paper_1707_02000_b200/csrc/build.cu paper_1707_02000_b200/csrc/capi.cu; make -s -C paper_1707_02000_b200/csrc -j16 2>&1 | grep error
