# Real-A DMMA shape variants (exploration) -> paper_1801_01434_b200/_variants/
#   BU (k extent per block row, uniform path), CT (8-output tiles per warp), MINB (min CTAs/SM, uniform path), SEG (amplitudes per exact re-seed),
#   PIPE (2-set block pipeline), GREC (G fragments by recurrence), NACC (accumulator sets by k-step parity),
#   W (consumer warps per CTA, uniform path)
set -e
cd "$(dirname "$0")/.."
mkdir -p paper_1801_01434_b200/_variants
rm -f paper_1801_01434_b200/_variants/*.so
build_one() {
  tag=BU$1_CT$2_MINB$3_SEG$4_PIPE$5_GREC$6_NACC$7_W$8
  out=paper_1801_01434_b200/_variants/libshorb200_$tag.so
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC \
    -DSHB_MMA_BU=$1 -DSHB_MMA_CT=$2 -DSHB_MMA_MINB_U=$3 -DSHB_MMA_SEG=$4 -DSHB_MMA_PIPE=$5 -DSHB_MMA_GREC=$6 -DSHB_MMA_NACC=$7 -DSHB_MMA_WARPS_U=$8 \
    -I include -c paper_1801_01434_b200/csrc/dft.cu -o /tmp/mrv_dft_$tag.o -Xptxas -v 2> /tmp/mrv_$tag.ptxas
  objs="/tmp/mrv_dft_$tag.o"
  for src in capi modexp collapse sample context dft_tc05; do objs="$objs paper_1801_01434_b200/_obj/$src.o"; done
  nvcc -gencode arch=compute_100a,code=sm_100a -shared $objs -o $out -lcudart
  echo "built $out: $(grep -A2 'dft_mma_kernelILb1ELb1' /tmp/mrv_$tag.ptxas | grep -oE 'Used [0-9]+ registers|[0-9]+ bytes spill stores' | tr '\n' ' ')"
}
for v in "128 1 1 32768 1 1 1 8" "128 1 1 32768 1 1 2 8" "112 1 1 32768 1 1 1 8" "128 1 1 65536 0 1 1 8"; do
  build_one $v &
done
wait
