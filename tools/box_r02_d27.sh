# width of the levels of >= 9000-row HSS fronts under stream priorities
mkdir -p gpurun_out
run() { tag=$1; shift; env "$@" timeout 900 python bench.py --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/d27_bench_$tag.json 2> gpurun_out/d27_bench_$tag.err; echo "bench $tag rc=$?"; python -c "
import json
d=json.loads(open('gpurun_out/d27_bench_$tag.json').read().strip().splitlines()[-1]); print('$tag', d['value'], d['e2e']['value'], d['relres'])"; tail -n 2 gpurun_out/d27_bench_$tag.err; }
run big6 A=1
run big5 HSSMF_HSS_STREAMS_BIG=5
run big7 HSSMF_HSS_STREAMS_BIG=7
run big8 HSSMF_HSS_STREAMS_BIG=8
run big3 HSSMF_HSS_STREAMS_BIG=3
