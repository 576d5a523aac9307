# validation after the last host-side change (no host copy of the matrix in analyze)
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -x -q > gpurun_out/d19_tests.txt 2>&1; echo "tests rc=$?"; tail -n 3 gpurun_out/d19_tests.txt
HSSMF_DEBUG_AN=1 timeout 1200 python bench.py > gpurun_out/d19_bench_full.json 2> gpurun_out/d19_bench_full.err; echo "full bench rc=$?"; grep analyze gpurun_out/d19_bench_full.err | tail -n 2
python - <<'P'
import json
d = json.loads(open("gpurun_out/d19_bench_full.json").read().strip().splitlines()[-1]); print(d["value"], d["e2e"]["value"], d.get("relres"), (d.get("roofline") or {}).get("frac"))
P
