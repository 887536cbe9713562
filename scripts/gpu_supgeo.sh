# Support-pass block geometry: forced small / forced big / chosen on the device, per config.
mkdir -p gpurun_out
for c in ${CFGS:-5 3 4 1}; do
  for f in 0 1 auto; do
    if [ $f = auto ]; then unset TDG_SUP_BIG; else export TDG_SUP_BIG=$f; fi
    TDG_SUP_DEBUG=1 timeout 900 python scripts/run_one.py $c 2 > gpurun_out/geo_${f}_c$c.log 2>&1
    echo "c$c force=$f: $(grep 'tdg support' gpurun_out/geo_${f}_c$c.log | tail -1) $(tail -1 gpurun_out/geo_${f}_c$c.log | grep -o 'parity=[a-zA-Z]*') $(tail -1 gpurun_out/geo_${f}_c$c.log | grep -o "'support_ms[^,]*")"
  done
done
unset TDG_SUP_BIG
