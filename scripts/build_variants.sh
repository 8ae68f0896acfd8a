# Build libshorb200 variants (exploration only) into paper_1801_01434_b200/_variants/
set -e
cd "$(dirname "$0")/.."
mkdir -p paper_1801_01434_b200/_variants
for v in "256 4" "256 2" "128 4" "128 8" "512 2"; do
  set -- $v
  out=paper_1801_01434_b200/_variants/libshorb200_T$1_K$2.so
  objs=""
  for src in capi modexp collapse dft dft_tc05 sample context; do
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC \
      -DSHB_DFT_THREADS=$1 -DSHB_DFT_K64=$2 -I include -c paper_1801_01434_b200/csrc/$src.cu \
      -o /tmp/var_$src.o
    objs="$objs /tmp/var_$src.o"
  done
  nvcc -gencode arch=compute_100a,code=sm_100a -shared $objs -o $out -lcudart
  echo built $out
done
