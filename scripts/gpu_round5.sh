mkdir -p gpurun_out
python -m paper_1801_01434_b200.build > gpurun_out/build.log 2>&1; echo build=$?
make -s -C oracle
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu.log
SHB_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 --modulus 3127 --seed 0 --steps 2 --warmup 3 > gpurun_out/bench_2rank_gloo.json 2> gpurun_out/bench_2rank_gloo.err; echo bench2=$?
cat gpurun_out/bench_2rank_gloo.json; tail -5 gpurun_out/bench_2rank_gloo.err
timeout 900 python scripts/configs_table.py --skip-46927 > gpurun_out/configs_table.jsonl 2> gpurun_out/configs_table.err; echo table=$?
cat gpurun_out/configs_table.jsonl; tail -3 gpurun_out/configs_table.err
