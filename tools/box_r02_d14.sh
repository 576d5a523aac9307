# device block list across engines, position maps by merge: full GPU suite, e2e with and without the list
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -x -q > gpurun_out/d14_tests.txt 2>&1; echo "tests rc=$?"; tail -n 4 gpurun_out/d14_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/d14_smoke.txt 2>&1; echo "smoke rc=$?"; tail -n 2 gpurun_out/d14_smoke.txt
run() { tag=$1; shift; env "$@" timeout 900 python bench.py --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/d14_bench_$tag.json 2> gpurun_out/d14_bench_$tag.err; echo "bench $tag rc=$?"; python -c "
import json
d=json.loads(open('gpurun_out/d14_bench_$tag.json').read().strip().splitlines()[-1]); print('$tag', d['value'], d['e2e']['value'], d['relres'])"; grep "analyze" gpurun_out/d14_bench_$tag.err | tail -n 3; }
run cache HSSMF_DEBUG_AN=1
run nocache HSSMF_NO_DEV_CACHE=1
run cache2 A=1
run lanes_gemm HSSMF_LANES=1
run lanes_all HSSMF_LANES=all
