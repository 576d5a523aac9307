# BASELINE configs 1-4 with the final build (types, ranks, relres against the reference goldens)
mkdir -p gpurun_out
for c in c1 c2 c3 c4; do
  timeout 900 python tools/run_config.py $c >> gpurun_out/d21_configs_c1_c4.jsonl 2>> gpurun_out/d21_configs.err; echo "$c rc=$?"
done
cat gpurun_out/d21_configs_c1_c4.jsonl | cut -c1-700
