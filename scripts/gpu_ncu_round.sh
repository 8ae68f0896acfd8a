mkdir -p gpurun_out
python -m paper_1801_01434_b200.build > gpurun_out/build.log 2>&1; echo build=$?
make -s -C oracle
# 1) launch list of the default bench command (plain run first, same command)
timeout 900 python bench.py > gpurun_out/bench_plain.json 2> gpurun_out/bench_plain.err && \
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_default.csv python bench.py > gpurun_out/ncu_launches_default.log 2>&1; echo ncu_launches=$?
cat gpurun_out/bench_plain.json
# 2) full-set captures at q=2^24 of the current uniform and generic kernels
timeout 600 python scripts/dft_paths_timing.py > gpurun_out/dft_paths2.json 2> gpurun_out/dft_paths2.err && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:dft_kernel -c 2 -o gpurun_out/dft_paths_full python scripts/dft_paths_timing.py > gpurun_out/ncu_paths_full.log 2>&1; echo ncu_full=$?
tail -3 gpurun_out/ncu_paths_full.log
cat gpurun_out/dft_paths2.json
