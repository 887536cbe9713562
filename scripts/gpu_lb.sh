# sweep the peel's min-blocks-per-SM launch bound (registers vs occupancy)
for b in 4 5 6; do
  make -s -C paper_1707_02000_b200/csrc clean >/dev/null; make -s -C paper_1707_02000_b200/csrc -j16 NVEXTRA="-DTDG_PEEL_MINB=$b" 2>&1 | grep -E "error" 
  for c in 3 5; do echo "minb=$b"; timeout 900 python scripts/run_one.py $c 2 2>&1 | tail -1; done
done
