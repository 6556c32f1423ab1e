# build libbnff_<tag>.so variants of the working tree with extra nvcc defines for every .cu:
#   tools/ab_macro.sh A "-DBNFF_TF32_STACK=0" B ""
set -e
cd "$(dirname "$0")/.."
python __graft_entry__.py > /dev/null
while [ $# -gt 1 ]; do
  tag=$1; defs=$2; shift 2
  objs=""
  for f in paper_1807_01702_b200/csrc/*.cu; do
    b=$(basename $f .cu)
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -diag-suppress 177 $defs -c -o build/${b}_$tag.o $f &
    objs="$objs build/${b}_$tag.o"
  done
  wait
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_1807_01702_b200/libbnff_$tag.so $objs
  echo built $tag
done
