# Peel regression bisect over round-2 commits (each tree built in bisect/<sha>, git-ignored).
mkdir -p gpurun_out
for c in 85a0c40 d075d6a bd49816 5361099 80e79c4 791d9e7 b185060; do
  (cd bisect/$c && timeout 600 python scripts/run_one.py 5 2 > ../../gpurun_out/bis_$c.log 2>&1; echo "$c rc=$?"; tail -1 ../../gpurun_out/bis_$c.log)
done
timeout 600 python scripts/run_one.py 5 2 > gpurun_out/bis_head.log 2>&1; echo "head rc=$?"; tail -1 gpurun_out/bis_head.log
