# int8 tensor-core FP64 DFT variants (exploration) -> paper_1801_01434_b200/_variants/
#   VARIANTS: lines "name -Dflags..." compiled into dft_i8.cu (e.g. "trace -DSHB_I8_TRACE")
set -e
cd "$(dirname "$0")/.."
mkdir -p paper_1801_01434_b200/_variants
rm -f paper_1801_01434_b200/_variants/*.so
DEFAULT_VARIANTS="trace -DSHB_I8_TRACE"
while read -r name flags; do
  [ -z "$name" ] && continue
  out=paper_1801_01434_b200/_variants/libshorb200_i8_$name.so
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC \
    $flags -I include -c paper_1801_01434_b200/csrc/dft_i8.cu -o /tmp/i8_$name.o
  objs="/tmp/i8_$name.o"
  for src in capi modexp collapse dft dft_tc05 sample context gates; do objs="$objs paper_1801_01434_b200/_obj/$src.o"; done
  nvcc -gencode arch=compute_100a,code=sm_100a -shared $objs -o $out -lcudart
  echo built $out
done <<< "${VARIANTS:-$DEFAULT_VARIANTS}"
