mkdir -p gpurun_out
python -m paper_1801_01434_b200.build > gpurun_out/build.log 2>&1; echo build=$?
timeout 600 ./scripts/dft_sweep > gpurun_out/dft_sweep.log 2>&1; echo sweep=$?
cat gpurun_out/dft_sweep.log
for cfg in "32399 2" "32399 0" "46927 0"; do
  timeout 1500 python scripts/run_config.py $cfg >> gpurun_out/traces_large.jsonl 2>> gpurun_out/traces_large.err; echo "cfg $cfg rc=$?"
done
cat gpurun_out/traces_large.jsonl; tail -3 gpurun_out/traces_large.err
