# width of the levels of small HSS fronts (< 9000 rows) under stream priorities
mkdir -p gpurun_out
run() { tag=$1; shift; env "$@" timeout 900 python bench.py --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/d20_bench_$tag.json 2> gpurun_out/d20_bench_$tag.err; echo "bench $tag rc=$?"; python -c "
import json
d=json.loads(open('gpurun_out/d20_bench_$tag.json').read().strip().splitlines()[-1]); print('$tag', d['value'], d['e2e']['value'], d['relres'])"; tail -n 2 gpurun_out/d20_bench_$tag.err; }
run base A=1
run small12 HSSMF_HSS_STREAMS_SMALL=12
run small16 HSSMF_HSS_STREAMS_SMALL=16
run small6 HSSMF_HSS_STREAMS_SMALL=6
