mkdir -p gpurun_out
python -m paper_1801_01434_b200.build > gpurun_out/build.log 2>&1; echo build=$?
make -s -C oracle
timeout 600 ./scripts/dft_sweep > gpurun_out/dft_sweep.log 2>&1; echo sweep=$?
cat gpurun_out/dft_sweep.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_default2.json 2> gpurun_out/bench_default2.err; echo bench=$?
cat gpurun_out/bench_default2.json; tail -3 gpurun_out/bench_default2.err
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-factoring --no-fp32"
timeout 600 $CMD > gpurun_out/plain_q30.json 2> gpurun_out/plain_q30.err && \
timeout 900 ncu --clock-control none -k regex:dft_kernel -c 1 --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --csv --log-file gpurun_out/dft_q30_metrics.csv $CMD > gpurun_out/ncu_q30.log 2>&1; echo ncu_q30=$?
cat gpurun_out/dft_q30_metrics.csv | tail -8
for cfg in "32399 2" "32399 0"; do
  timeout 900 python scripts/run_config.py $cfg >> gpurun_out/traces_large.jsonl 2>> gpurun_out/traces_large.err; echo "cfg $cfg rc=$?"
done
cat gpurun_out/traces_large.jsonl; tail -3 gpurun_out/traces_large.err
