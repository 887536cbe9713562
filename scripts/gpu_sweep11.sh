# support: table load factor (slots per key) and blocks/SM
summ() { python -c "
import sys,ast
for l in sys.stdin:
    if not l.startswith('C') or '{' not in l: continue
    d=ast.literal_eval(l[l.index('{'):])
    print({k:d.get(k) for k in ('build_ms','support_ms','peel_ms','process_ms','total_ms')})"; }
IFS=';' read -ra VS <<< "${VARIANTS:-load2:;load4:-DTDG_SUP_LOAD=4;load4m5:-DTDG_SUP_LOAD=4 -DTDG_SUP_MINB=5;load2m5:-DTDG_SUP_MINB=5}"
for v in "${VS[@]}"; do
  name="${v%%:*}"; flags="${v#*:}"
  touch paper_1707_02000_b200/csrc/*.cu; make -s -C paper_1707_02000_b200/csrc -j16 NVEXTRA="$flags" 2>&1 | grep -E "error"
  for c in ${CONFIGS:-3 5}; do echo "== $name C$c"; timeout 240 python scripts/run_one.py $c 2 2>&1 | summ; done
done
touch paper_1707_02000_b200/csrc/*.cu; make -s -C paper_1707_02000_b200/csrc -j16 2>&1 | grep error
