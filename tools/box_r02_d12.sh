# width of the concurrent HSS fronts under stream priorities; full default bench lines (ours + reference arm)
mkdir -p gpurun_out
run() { tag=$1; shift; env "$@" timeout 900 python bench.py --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/d12_bench_$tag.json 2> gpurun_out/d12_bench_$tag.err; echo "bench $tag rc=$?"; python -c "
import json
d=json.loads(open('gpurun_out/d12_bench_$tag.json').read().strip().splitlines()[-1]); print('$tag', d['value'], d['e2e']['value'], d['relres'])"; tail -n 2 gpurun_out/d12_bench_$tag.err; }
run w4 HSSMF_HSS_STREAMS=4
run w8 HSSMF_HSS_STREAMS=8
run w12 HSSMF_HSS_STREAMS=12
run specfold HSSMF_SPEC_FOLD=1
timeout 1200 python bench.py > gpurun_out/d12_bench_full.json 2> gpurun_out/d12_bench_full.err; echo "full bench rc=$?"; tail -c 400 gpurun_out/d12_bench_full.json
timeout 900 python bench.py --impl reference > gpurun_out/d12_bench_ref.json 2> gpurun_out/d12_bench_ref.err; echo "ref bench rc=$?"; tail -c 600 gpurun_out/d12_bench_ref.json
