# peel knobs: probe chains per lane (U) x min blocks/SM, bucket-sort threshold
summ() { python -c "
import sys,ast
for l in sys.stdin:
    if not l.startswith('C') or '{' not in l: continue
    d=ast.literal_eval(l[l.index('{'):])
    print({k:d[k] for k in ('support_ms','peel_ms','scan_ms','process_ms','compact_ms','total_ms')})"; }
IFS=';' read -ra VS <<< "${VARIANTS:-base:;u4m3:-DTDG_PEEL_U=4 -DTDG_PEEL_MINB=3;u4m2:-DTDG_PEEL_U=4 -DTDG_PEEL_MINB=2;u3m4:-DTDG_PEEL_U=3;s256k:-DTDG_SORT_MIN=262144;s64k:-DTDG_SORT_MIN=65536}"
for v in "${VS[@]}"; do
  name="${v%%:*}"; flags="${v#*:}"
  touch paper_1707_02000_b200/csrc/peel.cu; make -s -C paper_1707_02000_b200/csrc -j16 NVEXTRA="$flags" 2>&1 | grep -E "error"
  for c in ${CONFIGS:-3 5}; do echo "== $name C$c"; timeout 600 python scripts/run_one.py $c 2 2>&1 | summ; done
done
touch paper_1707_02000_b200/csrc/peel.cu; make -s -C paper_1707_02000_b200/csrc -j16 2>&1 | grep error
touch paper_1707_02000_b200/csrc/support.cu; make -s -C paper_1707_02000_b200/csrc -j16 NVEXTRA=-DTDG_SUP_TAB=2048 2>&1 | grep error
for c in ${CONFIGS:-3 5}; do echo "== suptab2048 C$c"; timeout 600 python scripts/run_one.py $c 2 2>&1 | summ; done
touch paper_1707_02000_b200/csrc/support.cu; make -s -C paper_1707_02000_b200/csrc -j16 2>&1 | grep error
