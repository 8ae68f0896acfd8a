# What the driver runs at round end, on one GPU (through gpurun):
#   build(), pytest -m gpu, smoke(), bench.py (driver flags), bench.py --impl reference,
#   and the ncu launch list of a short bench run (per-launch times, cold and serialised).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
tail -1 gpurun_out/smoke.log
timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo bench=$?
tail -3 gpurun_out/bench_final.err
timeout 1500 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_ref_final.json 2> gpurun_out/bench_ref_final.err; echo ref=$?
[ -n "$SHB_NCU" ] || exit 0
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 1 --no-factoring --no-cpu-baseline --no-dmma --no-e2e > gpurun_out/ncu_bench.log 2>&1; echo ncu=$?
