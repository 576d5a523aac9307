# determinism of the Householder route on c4 (and the Gram route on c3) under the concurrency knobs
mkdir -p gpurun_out
{
timeout 600 python tools/determinism.py c4 --repeat 3
HSSMF_LEVEL_PASS=1 timeout 600 python tools/determinism.py c4 --repeat 2
HSSMF_NO_SPEC_SAMPLING=1 timeout 600 python tools/determinism.py c4 --repeat 2
HSSMF_HSS_STREAMS=1 timeout 900 python tools/determinism.py c4 --repeat 2
HSSMF_NO_TMA=1 timeout 600 python tools/determinism.py c4 --repeat 2
timeout 600 python tools/determinism.py c3 --repeat 3
} > gpurun_out/d6_determinism.txt 2>&1
cat gpurun_out/d6_determinism.txt
timeout 900 python bench.py --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/d6_bench.json 2> gpurun_out/d6_bench.err; echo "bench rc=$?"
HSSMF_ID_SOLVE=subst timeout 900 python bench.py --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/d6_bench_subst.json 2> gpurun_out/d6_bench_subst.err; echo "bench subst rc=$?"
python - <<'P'
import json
for t in ("d6_bench", "d6_bench_subst"):
    d = json.loads(open(f"gpurun_out/{t}.json").read().strip().splitlines()[-1]); print(t, d["value"], d["e2e"]["value"], d["relres"])
P
