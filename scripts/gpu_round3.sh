mkdir -p gpurun_out
python -m paper_1801_01434_b200.build > gpurun_out/build.log 2>&1; echo build=$?
make -s -C oracle
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/bench_default3.json 2> gpurun_out/bench_default3.err; echo bench=$?
cat gpurun_out/bench_default3.json; tail -3 gpurun_out/bench_default3.err
timeout 1500 python scripts/run_config.py 46927 0 >> gpurun_out/traces_large.jsonl 2>> gpurun_out/traces_large.err; echo "cfg 46927 rc=$?"
tail -1 gpurun_out/traces_large.jsonl; tail -3 gpurun_out/traces_large.err
