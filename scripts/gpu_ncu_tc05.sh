# ncu evidence for the tcgen05 FP32 kernel: --set full at q = 2^24 and 2^30
mkdir -p gpurun_out
python -m paper_1801_01434_b200.build > gpurun_out/build.log 2>&1; echo build=$?
timeout 300 python scripts/tc05_once.py > gpurun_out/tc05_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dft_tc05 -c 2 -o gpurun_out/dft_tc05_full2 python scripts/tc05_once.py > gpurun_out/ncu_tc05.log 2>&1; echo ncu=$?
tail -2 gpurun_out/ncu_tc05.log
