# sweep a compile-time knob: VARIANTS="name:flags;name:flags" ; CONFIGS ; counters on
IFS=';' read -ra VS <<< "$VARIANTS"
for v in "${VS[@]}"; do
  name="${v%%:*}"; flags="${v#*:}"
  touch paper_1707_02000_b200/csrc/peel.cu; make -s -C paper_1707_02000_b200/csrc -j16 NVEXTRA="$flags" 2>&1 | grep -E "error"
  for c in ${CONFIGS:-3}; do echo "== $name C$c"; TDG_COUNT_HITS=${COUNT:-0} timeout 900 python scripts/run_one.py $c ${REPS:-1} 2>&1 | tail -1 | python -c "
import sys,ast
l=sys.stdin.read(); d=ast.literal_eval(l[l.index('{'):])
print({k:d[k] for k in ('support_ms','peel_ms','scan_ms','process_ms','compact_ms','total_ms','probes','support_probes','hits','dead_probes','compactions')})"; done
done
