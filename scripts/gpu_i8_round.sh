# int8 FP64 engine as the default: GPU tests, smoke, bench, ncu evidence
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_i8.json 2> gpurun_out/bench_i8.err; echo bench=$?
cat gpurun_out/bench_i8.json; tail -3 gpurun_out/bench_i8.err
[ -n "$NO_NCU" ] && exit 0
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_i8.csv \
  python bench.py --steps 2 --warmup 3 --no-dmma > gpurun_out/ncu_launches_i8.log 2>&1; echo launches=$?
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active,smsp__mem_tensor_reads_op_ldt.sum.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed \
  --clock-control none --csv -k regex:dft_i8 python scripts/i8_once.py big > gpurun_out/i8_q30_metrics.csv 2> gpurun_out/i8_q30_metrics.err; echo metrics=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dft_i8 -c 1 -o gpurun_out/dft_i8_final python scripts/i8_once.py > gpurun_out/ncu_i8_final.log 2>&1; echo ncu=$?
