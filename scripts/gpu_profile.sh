mkdir -p gpurun_out
python -m paper_1801_01434_b200.build > gpurun_out/build.log 2>&1; echo build=$?
make -s -C oracle
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python scripts/step_breakdown.py 32399 8 > gpurun_out/breakdown.log 2>&1; echo breakdown=$?
cat gpurun_out/breakdown.log
CMD="python bench.py --modulus 3127 --seed 0 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-factoring"
timeout 600 $CMD > gpurun_out/plain_3127.json 2> gpurun_out/plain_3127.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_3127.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo ncu_launches=$?
cat gpurun_out/plain_3127.json
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:dft_kernel -c 1 -o gpurun_out/dft_uniform_3127 $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu_full=$?
tail -3 gpurun_out/ncu_full.log
ls -la gpurun_out
