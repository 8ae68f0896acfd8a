mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
python -m paper_1801_01434_b200.build > gpurun_out/build.log 2>&1; echo build=$?
make -s -C oracle
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -30 gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo smoke=$?
tail -3 gpurun_out/smoke.log
timeout 600 python bench.py --modulus 3127 --seed 0 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_3127.json 2> gpurun_out/bench_3127.err; echo bench3127=$?
cat gpurun_out/bench_3127.json; tail -5 gpurun_out/bench_3127.err
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo benchfull=$?
cat gpurun_out/bench_full.json; tail -5 gpurun_out/bench_full.err
