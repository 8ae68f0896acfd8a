mkdir -p gpurun_out
python -m paper_1801_01434_b200.build > gpurun_out/build.log 2>&1; echo build=$?
make -s -C oracle
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench=$?
cat gpurun_out/bench_default.json; tail -3 gpurun_out/bench_default.err
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-factoring"
timeout 600 $CMD > gpurun_out/plain_full.json 2> gpurun_out/plain_full.err && \
timeout 2700 ncu --set full --clock-control none --import-source on -k regex:dft_kernel -c 1 -o gpurun_out/dft_uniform_q2_30 $CMD > gpurun_out/ncu_full_q30.log 2>&1; echo ncu_full=$?
tail -3 gpurun_out/ncu_full_q30.log
