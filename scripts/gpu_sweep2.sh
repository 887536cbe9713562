# A/B: support lookup form (TDG_SUP_HASH) at C3/C5, then peel staging thresholds.
summ() { python -c "
import sys,ast
for l in sys.stdin:
    if not l.startswith('C') or '{' not in l: continue
    d=ast.literal_eval(l[l.index('{'):])
    print({k:d[k] for k in ('support_ms','peel_ms','scan_ms','process_ms','compact_ms','total_ms','probes','support_probes')})"; }
for c in ${CONFIGS:-3 5}; do
  for h in 0 1; do echo "== SUP_HASH=$h C$c"; TDG_SUP_HASH=$h timeout 600 python scripts/run_one.py $c 2 2>&1 | summ; done
done
IFS=';' read -ra VS <<< "${VARIANTS:-m512r8:-DTDG_STAGE_MIN=512;m128r8:-DTDG_STAGE_MIN=128;m64r32:-DTDG_STAGE_MIN=64 -DTDG_STAGE_RATIO=32;off:-DTDG_STAGE_MIN=0}"
for v in "${VS[@]}"; do
  name="${v%%:*}"; flags="${v#*:}"
  touch paper_1707_02000_b200/csrc/peel.cu; make -s -C paper_1707_02000_b200/csrc -j16 NVEXTRA="$flags" 2>&1 | grep -E "error"
  for c in ${CONFIGS:-3 5}; do echo "== $name C$c"; timeout 600 python scripts/run_one.py $c 2 2>&1 | summ; done
done
touch paper_1707_02000_b200/csrc/peel.cu; make -s -C paper_1707_02000_b200/csrc -j16 2>&1 | grep error
