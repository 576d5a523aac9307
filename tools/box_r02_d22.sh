# shorter TMA sampling CTAs (more split-K slices) so that SMs return to the other fronts' chains sooner
mkdir -p gpurun_out
run() { tag=$1; shift; env "$@" timeout 900 python bench.py --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/d22_bench_$tag.json 2> gpurun_out/d22_bench_$tag.err; echo "bench $tag rc=$?"; python -c "
import json
d=json.loads(open('gpurun_out/d22_bench_$tag.json').read().strip().splitlines()[-1]); print('$tag', d['value'], d['e2e']['value'], d['relres'])"; tail -n 2 gpurun_out/d22_bench_$tag.err; }
run base A=1
run k2048 HSSMF_SPLITK_KSLICE=2048
run k1024 HSSMF_SPLITK_KSLICE=1024
run k512 HSSMF_SPLITK_KSLICE=512
run base2 A=1
