# tcgen05 FP32 DFT variants (exploration) -> paper_1801_01434_b200/_variants/
#   BK: k per row-block (128: one G buffer; 64: G double-buffered, built under the MMAs)
#   CH: Horner chains in the fold (1 of 64 row-blocks, or 4 of 16)
set -e
cd "$(dirname "$0")/.."
mkdir -p paper_1801_01434_b200/_variants
rm -f paper_1801_01434_b200/_variants/*.so
for v in ${VARIANTS:-"64 4" "128 4" "64 1"}; do
  set -- $v
  bk=$1
  out=paper_1801_01434_b200/_variants/libshorb200_tc05_BK$1_CH$2.so
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC \
    -DSHB_TC05_BK=$1 -DSHB_TC05_CHAINS=$2 -I include -c paper_1801_01434_b200/csrc/dft_tc05.cu -o /tmp/tc05_$bk.o
  objs="/tmp/tc05_$bk.o"
  for src in capi modexp collapse dft sample context; do objs="$objs paper_1801_01434_b200/_obj/$src.o"; done
  nvcc -gencode arch=compute_100a,code=sm_100a -shared $objs -o $out -lcudart
  echo built $out
done
