mkdir -p gpurun_out
python -m paper_1801_01434_b200.build > gpurun_out/build.log 2>&1; echo build=$?
make -s -C oracle
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python scripts/dft_paths_timing.py > gpurun_out/dft_paths3.json 2> gpurun_out/dft_paths3.err; echo paths=$?
cat gpurun_out/dft_paths3.json; tail -3 gpurun_out/dft_paths3.err
