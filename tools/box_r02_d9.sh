# c4 (Householder route) run-to-run determinism by knob, 4 runs each; compute-sanitizer on the small driver
mkdir -p gpurun_out
{
for v in "A=1" "HSSMF_NO_TMA=1" "HSSMF_GEMM_NO_SMALL=1" "HSSMF_CPQR_CLUSTER=1" "HSSMF_LEVEL_PASS=1"; do
  env $v timeout 900 python tools/determinism.py c4 --repeat 4 2>&1 | grep "^c4" | sed "s/^/[$v] /"
done
} > gpurun_out/d9_c4_determinism.txt 2>&1
cat gpurun_out/d9_c4_determinism.txt
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool python tools/sanitize_small.py > gpurun_out/d9_sanitizer_$tool.txt 2>&1; echo "$tool rc=$?"
  tail -n 4 gpurun_out/d9_sanitizer_$tool.txt
done
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/d9_bench.json 2> gpurun_out/d9_bench.err; echo "bench rc=$?"
python -c "
import json
d=json.loads(open('gpurun_out/d9_bench.json').read().strip().splitlines()[-1]); print('bench', d['value'], d['e2e']['value'], d['relres'], d['roofline']['frac'])"
