# Build A/B variants of libtdg.so with compile-time knobs (measurement only):
#   bash scripts/variants.sh name1 "-DKNOB=1 -DOTHER=2" name2 "-DKNOB=3" ...
# -> paper_1707_02000_b200/lib_variants/<name>/libtdg.so ; select with TDG_SO=<path> at run time.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  out=$ROOT/paper_1707_02000_b200/lib_variants/$name
  mkdir -p $out
  make -s -C $ROOT/paper_1707_02000_b200/csrc -j8 LIB=$out NVEXTRA="$flags" $out/libtdg.so
  echo "built $name ($flags)"
done
