# dependency-driven schedule for the top tree levels only (HSSMF_REGION_LEVEL=k)
mkdir -p gpurun_out
run() { tag=$1; shift; env "$@" timeout 900 python bench.py --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/d18_bench_$tag.json 2> gpurun_out/d18_bench_$tag.err; echo "bench $tag rc=$?"; python -c "
import json
d=json.loads(open('gpurun_out/d18_bench_$tag.json').read().strip().splitlines()[-1]); print('$tag', d['value'], d['e2e']['value'], d['relres'])"; tail -n 2 gpurun_out/d18_bench_$tag.err; }
run base A=1
run top2 HSSMF_REGION_LEVEL=2
run top3 HSSMF_REGION_LEVEL=3
run top4 HSSMF_REGION_LEVEL=4
run base2 A=1
