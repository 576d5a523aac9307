# last validation of the final build: kernel + spec tests (new transposed-TMA test), default bench line
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -x -q > gpurun_out/d17_tests.txt 2>&1; echo "tests rc=$?"; tail -n 3 gpurun_out/d17_tests.txt
timeout 1200 python bench.py > gpurun_out/d17_bench_full.json 2> gpurun_out/d17_bench_full.err; echo "full bench rc=$?"
python - <<'P'
import json
d = json.loads(open("gpurun_out/d17_bench_full.json").read().strip().splitlines()[-1]); print(d["value"], d["e2e"]["value"], d.get("relres"), (d.get("roofline") or {}).get("frac"))
for r in d.get("rooflines") or []: print("   ", r["kernel"], r.get("bound"), round(r.get("achieved", 0), 1), r.get("unit"), round(r.get("frac", 0), 3) if r.get("frac") else None)
P
