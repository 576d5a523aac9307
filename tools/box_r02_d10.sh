# stream priorities: worker streams high, big kernels through low-priority lanes
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_spec.py tests/test_gpu_hss.py tests/test_gpu_mf.py -x -q > gpurun_out/d10_tests.txt 2>&1; echo "tests rc=$?"; tail -n 3 gpurun_out/d10_tests.txt
run() { tag=$1; shift; env "$@" timeout 900 python bench.py --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/d10_bench_$tag.json 2> gpurun_out/d10_bench_$tag.err; echo "bench $tag rc=$?"; python -c "
import json
d=json.loads(open('gpurun_out/d10_bench_$tag.json').read().strip().splitlines()[-1]); print('$tag', d['value'], d['e2e']['value'], d['relres'])"; tail -n 2 gpurun_out/d10_bench_$tag.err; }
run lanes A=1
run prio_only HSSMF_NO_LANES=1
run noprio HSSMF_NO_PRIO=1
run lanes2 A=1
run lanes_w8 HSSMF_HSS_STREAMS=8
HSSMF_DEBUG=1 timeout 900 python tools/gpu_fronts.py c5 --out gpurun_out/d10_dbg.npz > gpurun_out/d10_dbg.log 2>&1; grep "level:" gpurun_out/d10_dbg.log
