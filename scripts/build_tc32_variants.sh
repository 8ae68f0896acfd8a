# FP32 tensor-core (bf16x2) DFT variants (exploration) -> paper_1801_01434_b200/_variants/
#   BK (k extent per block row), MINB (min CTAs/SM), SEG (amplitudes per FP64 segment)
set -e
cd "$(dirname "$0")/.."
mkdir -p paper_1801_01434_b200/_variants
rm -f paper_1801_01434_b200/_variants/*.so
build_one() {
  tag=BK$1_MINB$2_SEG$3
  out=paper_1801_01434_b200/_variants/libshorb200_tc_$tag.so
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC \
    -DSHB_TC_BK=$1 -DSHB_TC_MINB=$2 -DSHB_TC_SEG=$3 \
    -I include -c paper_1801_01434_b200/csrc/dft.cu -o /tmp/tcv_dft_$tag.o -Xptxas -v 2> /tmp/tcv_$tag.ptxas
  objs="/tmp/tcv_dft_$tag.o"
  for src in capi modexp collapse sample context dft_tc05; do objs="$objs paper_1801_01434_b200/_obj/$src.o"; done
  nvcc -gencode arch=compute_100a,code=sm_100a -shared $objs -o $out -lcudart
  echo "built $out: $(grep -A2 'dft_tc32' /tmp/tcv_$tag.ptxas | grep -oE 'Used [0-9]+ registers|[0-9]+ bytes spill stores' | tr '\n' ' ')"
}
for v in ${VARIANTS:-"128 1 32768" "64 2 32768" "64 1 32768" "128 1 16384" "32 2 32768"}; do
  build_one $v &
done
wait
