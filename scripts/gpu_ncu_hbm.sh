mkdir -p gpurun_out
python -m paper_1801_01434_b200.build > gpurun_out/build.log 2>&1; echo build=$?
timeout 300 python scripts/hbm_kernels_once.py > gpurun_out/hbm_plain.log 2>&1 && \
timeout 1200 ncu --clock-control none -k regex:"modexp|class_counts|compact|geo" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed --csv --log-file gpurun_out/hbm_kernels.csv python scripts/hbm_kernels_once.py > gpurun_out/ncu_hbm.log 2>&1; echo ncu=$?
cat gpurun_out/hbm_plain.log; tail -2 gpurun_out/ncu_hbm.log
