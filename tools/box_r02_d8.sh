# warm-started IDs as a failure filter: parity (c3 node for node, c4 determinism), bench on/off, margins
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_spec.py -x -q > gpurun_out/d8_tests_a.txt 2>&1; echo "tests a rc=$?"; tail -n 3 gpurun_out/d8_tests_a.txt
HSSMF_DEBUG_ROUNDS=1 timeout 600 python tools/determinism.py c3 --repeat 2 > gpurun_out/d8_c3.txt 2>&1; grep "^c3" gpurun_out/d8_c3.txt; grep "warm" gpurun_out/d8_c3.txt | tail -n 3
timeout 600 python tools/determinism.py c4 --repeat 2 > gpurun_out/d8_c4.txt 2>&1; cat gpurun_out/d8_c4.txt
run() { tag=$1; shift; env "$@" timeout 900 python bench.py --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/d8_bench_$tag.json 2> gpurun_out/d8_bench_$tag.err; echo "bench $tag rc=$?"; python -c "
import json
d=json.loads(open('gpurun_out/d8_bench_$tag.json').read().strip().splitlines()[-1]); print('$tag', d['value'], d['e2e']['value'], d['relres'])"; tail -n 2 gpurun_out/d8_bench_$tag.err; }
run warm A=1
run cold HSSMF_WARM_IDS=0
run warm_m15 HSSMF_WARM_MARGIN=1.5
run warm_subst HSSMF_ID_SOLVE=subst
HSSMF_DEBUG_ROUNDS=1 timeout 900 python tools/gpu_fronts.py c5 --out gpurun_out/d8_c5_warm.npz > gpurun_out/d8_c5_warm.log 2>&1; grep warm gpurun_out/d8_c5_warm.log | tail -n 8; tail -n 1 gpurun_out/d8_c5_warm.log
timeout 1500 python -m pytest tests/test_gpu_hss.py tests/test_gpu_mf.py -x -q > gpurun_out/d8_tests_b.txt 2>&1; echo "tests b rc=$?"; tail -n 5 gpurun_out/d8_tests_b.txt
