# build libbnff_<tag>.so variants of the working tree with extra nvcc defines for wconv.cu:
#   tools/ab_defines.sh A "-DX=1" B "-DX=2" ...
set -e
cd "$(dirname "$0")/.."
python __graft_entry__.py > /dev/null
while [ $# -gt 1 ]; do
  tag=$1; defs=$2; shift 2
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -diag-suppress 177 $defs -c -o build/wconv_$tag.o paper_1807_01702_b200/csrc/wconv.cu
  objs=$(ls build/*.cu.o | grep -v wconv.cu.o)
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_1807_01702_b200/libbnff_$tag.so $objs build/wconv_$tag.o
  echo built $tag
done
