# wavefront ID batches, redux argmax, SYRK variants, region schedule: tests, microbench, A/B benches
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_spec.py tests/test_gpu_hss.py tests/test_gpu_mf.py -x -q > gpurun_out/d5_tests.txt 2>&1; echo "tests rc=$?"
tail -n 3 gpurun_out/d5_tests.txt
for v in dmma rmw rmw4; do
  HSSMF_GRAM_SYRK=$v timeout 200 python tools/gram_bench.py > gpurun_out/d5_gram_$v.json 2>&1; echo "gram $v rc=$?"
done
run() { tag=$1; shift; env "$@" timeout 900 python bench.py --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/d5_bench_$tag.json 2> gpurun_out/d5_bench_$tag.err; echo "bench $tag rc=$?"; python -c "
import json
d=json.loads(open('gpurun_out/d5_bench_$tag.json').read().strip().splitlines()[-1]); print('$tag', d['value'], d['e2e']['value'], d['relres'])"; }
run wave A=1
run level HSSMF_LEVEL_PASS=1
run rmw HSSMF_GRAM_SYRK=rmw
run rmw4 HSSMF_GRAM_SYRK=rmw4
run region HSSMF_REGION=1
run wave2 A=1
timeout 600 python tools/gemm_shapes_c5.py c5 > gpurun_out/d5_gemm_shapes_c5.txt 2>&1; echo "shapes rc=$?"
rm -f gpurun_out/probe_dump.csv
timeout 600 python tools/run_config.py c4 > gpurun_out/d5_c4.json 2> gpurun_out/d5_c4.err; echo "c4 rc=$?"; tail -c 600 gpurun_out/d5_c4.json
du -sh gpurun_out
