# large-config factoring traces on the default engines (SURVEY 8(d) expected traces)
mkdir -p gpurun_out
rm -f gpurun_out/traces_large.jsonl
for cfg in "32399 8" "32399 2" "32399 0" "32399 3" "46927 0"; do
  timeout 1200 python scripts/run_config.py $cfg >> gpurun_out/traces_large.jsonl 2>> gpurun_out/traces_large.err; echo "cfg $cfg rc=$?"
done
cat gpurun_out/traces_large.jsonl
