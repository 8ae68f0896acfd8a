# ncu metrics + timeline of the int8 DFT at the bench config and the launch list of a one-step bench (needs the trace build: VARIANTS="trace -DSHB_I8_TRACE" bash scripts/build_i8_variants.sh)
mkdir -p gpurun_out
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active
timeout 600 ncu --metrics $M --clock-control none -k regex:dft_i8_uniform -c 1 --csv python scripts/i8_once.py big2 > gpurun_out/k8_seed2_metrics.csv 2> gpurun_out/k8_seed2_metrics.err; echo ncu1=$?
TRACE_LIB=libshorb200_i8_trace.so SBA=32768 timeout 200 python scripts/i8_trace_run.py big2 > gpurun_out/tl_k8_big2.txt 2>&1; echo tl=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_k8.csv \
  python bench.py --steps 1 --warmup 1 --no-factoring --no-cpu-baseline --no-dmma --no-e2e > gpurun_out/ncu_bench_k8.log 2>&1; echo ncu2=$?
