# ncu evidence for the real-A DMMA DFT kernel (the bench's dominant kernel)
mkdir -p gpurun_out
python -m paper_1801_01434_b200.build > gpurun_out/build.log 2>&1; echo build=$?
make -s -C oracle
# 1) targeted metrics of the DFT launch at the bench config (q = 2^30)
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-factoring --no-fp32"
timeout 600 $CMD > gpurun_out/plain_q30.json 2> gpurun_out/plain_q30.err && \
timeout 900 ncu --clock-control none -k regex:dft_mma_kernel -c 1 --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --csv --log-file gpurun_out/dft_mma_q30_metrics.csv $CMD > gpurun_out/ncu_q30.log 2>&1; echo ncu_q30=$?
tail -8 gpurun_out/dft_mma_q30_metrics.csv
# 2) launch list of the default bench command (plain run first, same command)
timeout 900 python bench.py > gpurun_out/bench_plain.json 2> gpurun_out/bench_plain.err && \
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_default.csv python bench.py > gpurun_out/ncu_launches_default.log 2>&1; echo ncu_launches=$?
cat gpurun_out/bench_plain.json
# 3) full set of the uniform real-A kernel at q = 2^24
timeout 800 ncu --set full --clock-control none --import-source on -k regex:dft_mma_kernel --launch-skip 2 -c 1 -o gpurun_out/dft_mma_unif_real_full python scripts/mma_once.py > gpurun_out/ncu_full.log 2>&1; echo ncu_full=$?
tail -2 gpurun_out/ncu_full.log
