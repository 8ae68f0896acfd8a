mkdir -p gpurun_out
python -m paper_1801_01434_b200.build > gpurun_out/build.log 2>&1; echo build=$?
make -s -C oracle
SHB_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 --modulus 3127 --seed 0 --steps 2 --warmup 3 > gpurun_out/bench_2rank_gloo.json 2> gpurun_out/bench_2rank_gloo.err; echo bench2=$?
cat gpurun_out/bench_2rank_gloo.json; tail -5 gpurun_out/bench_2rank_gloo.err
SHB_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29556 bench.py --impl reference --gpus 2 --modulus 3127 --seed 0 --steps 1 --warmup 1 > gpurun_out/bench_2rank_ref.json 2> gpurun_out/bench_2rank_ref.err; echo benchref2=$?
cat gpurun_out/bench_2rank_ref.json; tail -3 gpurun_out/bench_2rank_ref.err
