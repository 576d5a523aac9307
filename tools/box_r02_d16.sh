# final validation of the round: full GPU suite, smoke, default bench (ours + reference arm)
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -x -q > gpurun_out/d16_tests.txt 2>&1; echo "tests rc=$?"; tail -n 3 gpurun_out/d16_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/d16_smoke.txt 2>&1; echo "smoke rc=$?"; tail -n 1 gpurun_out/d16_smoke.txt
timeout 900 python bench.py --impl reference > gpurun_out/d16_bench_ref.json 2> gpurun_out/d16_bench_ref.err; echo "ref bench rc=$?"
timeout 1200 python bench.py > gpurun_out/d16_bench_full.json 2> gpurun_out/d16_bench_full.err; echo "full bench rc=$?"
python - <<'P'
import json
for t in ("d16_bench_full", "d16_bench_ref"):
    d = json.loads(open(f"gpurun_out/{t}.json").read().strip().splitlines()[-1]); print(t, d["value"], d["e2e"]["value"], d.get("relres"), (d.get("roofline") or {}).get("frac"))
    for r in d.get("rooflines") or []: print("   ", r["kernel"], r.get("bound"), round(r.get("achieved", 0), 1), r.get("unit"), round(r.get("frac", 0), 3) if r.get("frac") else None)
P
