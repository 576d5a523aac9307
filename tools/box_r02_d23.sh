mkdir -p gpurun_out
timeout 900 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --gmres > gpurun_out/d23_bench_gmres.json 2> gpurun_out/d23_bench_gmres.err; echo "rc=$?"
python -c "
import json
d=json.loads(open('gpurun_out/d23_bench_gmres.json').read().strip().splitlines()[-1]); print(d['value'], d['relres'], d['gmres_preconditioned'])"
