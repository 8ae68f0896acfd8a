# int8 tensor-core FP64 DFT variants (exploration) -> paper_1801_01434_b200/_variants/
#   VARIANTS: lines "name -Dflags..." for dft_i8.cu (SHB_I8_NB, SHB_I8_BK, SHB_I8_ICOMB, ...)
set -e
cd "$(dirname "$0")/.."
mkdir -p paper_1801_01434_b200/_variants
rm -f paper_1801_01434_b200/_variants/*.so
DEFAULT_VARIANTS="nb32 -DSHB_I8_NB=32
fcomb -DSHB_I8_ICOMB=0
nb32fcomb -DSHB_I8_NB=32 -DSHB_I8_ICOMB=0"
while read -r name flags; do
  [ -z "$name" ] && continue
  out=paper_1801_01434_b200/_variants/libshorb200_i8_$name.so
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC \
    $flags -I include -c paper_1801_01434_b200/csrc/dft_i8.cu -o /tmp/i8_$name.o
  objs="/tmp/i8_$name.o"
  # the other digit count's engine comes from the default build (dft.cu links both)
  case "$flags" in *SHB_I8_DIGITS=6*) other=dft_i8 ;; *) other=dft_i8d6 ;; esac
  for src in capi modexp collapse dft dft_tc05 sample context $other; do objs="$objs paper_1801_01434_b200/_obj/$src.o"; done
  nvcc -gencode arch=compute_100a,code=sm_100a -shared $objs -o $out -lcudart
  echo built $out
done <<< "${VARIANTS:-$DEFAULT_VARIANTS}"
