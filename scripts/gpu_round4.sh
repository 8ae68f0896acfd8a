mkdir -p gpurun_out
python -m paper_1801_01434_b200.build > gpurun_out/build.log 2>&1; echo build=$?
make -s -C oracle
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python scripts/dft_paths_timing.py > gpurun_out/dft_paths.json 2> gpurun_out/dft_paths.err; echo paths=$?
cat gpurun_out/dft_paths.json; tail -3 gpurun_out/dft_paths.err
timeout 900 python bench.py > gpurun_out/bench_default4.json 2> gpurun_out/bench_default4.err; echo bench=$?
cat gpurun_out/bench_default4.json; tail -3 gpurun_out/bench_default4.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo benchref=$?
cat gpurun_out/bench_ref.json; tail -3 gpurun_out/bench_ref.err
