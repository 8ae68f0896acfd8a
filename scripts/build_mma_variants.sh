# DMMA-engine shape variants (exploration) -> paper_1801_01434_b200/_variants/
#   B (k extent per block row), CT (8-output tiles per warp), MINB (min CTAs/SM)
set -e
cd "$(dirname "$0")/.."
mkdir -p paper_1801_01434_b200/_variants
rm -f paper_1801_01434_b200/_variants/*.so
for v in ${VARIANTS:-"32 2 1" "32 1 1" "64 1 1" "16 2 1" "16 1 2"}; do
  set -- $v
  out=paper_1801_01434_b200/_variants/libshorb200_mmaB$1_CT$2_MINB$3.so
  objs=""
  for src in capi modexp collapse dft dft_tc05 sample context; do
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC \
      -DSHB_MMA_B=$1 -DSHB_MMA_CT=$2 -DSHB_MMA_MINB=$3 -I include -c paper_1801_01434_b200/csrc/$src.cu \
      -o /tmp/mv_$src.o 2>/dev/null
    objs="$objs /tmp/mv_$src.o"
  done
  nvcc -gencode arch=compute_100a,code=sm_100a -shared $objs -o $out -lcudart
  echo built $out
done
