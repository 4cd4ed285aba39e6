# Build experiment variants of the library (compile-time knobs) into _variants/<name>/.
# usage: tools/variants.sh name "-DKNOB=1 ..." [name2 "flags2" ...]
set -e
cd "$(dirname "$0")/.."
while [ $# -ge 2 ]; do
  d=_variants/$1
  mkdir -p $d
  EF_BUILD_OBJ=$d/obj EF_BUILD_OUT=$d/libedgeforge_b200.so EF_NVCC_EXTRA="$2" python -m paper_1710_07745_b200.build >/dev/null
  echo "built $d ($2)"
  shift 2
done
