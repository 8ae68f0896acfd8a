# int8 tensor-core FP64 DFT: variant timing + one ncu --set full capture at q = 2^24
mkdir -p gpurun_out
timeout 600 python scripts/i8_variant_timing.py ${BIG:-big} > gpurun_out/i8_variants.jsonl 2> gpurun_out/i8_variants.err; echo timing=$?
cat gpurun_out/i8_variants.jsonl
if [ -z "$NO_NCU" ]; then
timeout 300 python scripts/i8_once.py > gpurun_out/i8_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dft_i8 -c 1 -o gpurun_out/dft_i8_full python scripts/i8_once.py > gpurun_out/ncu_i8.log 2>&1; echo ncu=$?
tail -2 gpurun_out/ncu_i8.log
fi
