# TMA restricted to non-transposed operands: c4 determinism; transposed TMA GEMM repeatability; default bench; full GPU suite
mkdir -p gpurun_out
timeout 900 python tools/determinism.py c4 --repeat 4 2>&1 | grep "^c4" > gpurun_out/d11_c4_determinism.txt; cat gpurun_out/d11_c4_determinism.txt
HSSMF_TMA_TRANS=1 timeout 900 python tools/gemm_repro.py --repeat 6 > gpurun_out/d11_gemm_repro_trans.txt 2>&1; cat gpurun_out/d11_gemm_repro_trans.txt
run() { tag=$1; shift; env "$@" timeout 900 python bench.py --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/d11_bench_$tag.json 2> gpurun_out/d11_bench_$tag.err; echo "bench $tag rc=$?"; python -c "
import json
d=json.loads(open('gpurun_out/d11_bench_$tag.json').read().strip().splitlines()[-1]); print('$tag', d['value'], d['e2e']['value'], d['relres'])"; tail -n 2 gpurun_out/d11_bench_$tag.err; }
run default A=1
run tma_trans HSSMF_TMA_TRANS=1
run default2 A=1
timeout 3000 python -m pytest tests -m gpu -x -q > gpurun_out/d11_tests.txt 2>&1; echo "tests rc=$?"; tail -n 5 gpurun_out/d11_tests.txt
