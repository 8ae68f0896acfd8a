mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo bench=$?
cat gpurun_out/bench_final.json; tail -3 gpurun_out/bench_final.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_final.json 2> gpurun_out/bench_ref_final.err; echo ref=$?
cat gpurun_out/bench_ref_final.json
[ -n "$SHB_TRACES" ] || exit 0
rm -f gpurun_out/traces_large.jsonl
for cfg in "32399 8" "32399 2" "32399 0" "46927 0"; do
  timeout 1200 python scripts/run_config.py $cfg >> gpurun_out/traces_large.jsonl 2>> gpurun_out/traces_large.err; echo "cfg $cfg rc=$?"
done
cat gpurun_out/traces_large.jsonl
