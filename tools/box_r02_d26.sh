# last check of the committed state: full GPU suite, smoke, default bench
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -x -q > gpurun_out/d26_tests.txt 2>&1; echo "tests rc=$?"; tail -n 2 gpurun_out/d26_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/d26_smoke.txt 2>&1; echo "smoke rc=$?"; tail -n 1 gpurun_out/d26_smoke.txt
timeout 1200 python bench.py > gpurun_out/d26_bench_full.json 2> gpurun_out/d26_bench_full.err; echo "full bench rc=$?"
python -c "
import json
d=json.loads(open('gpurun_out/d26_bench_full.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['relres'], d['roofline']['frac'], d['gpu_launches'])"
