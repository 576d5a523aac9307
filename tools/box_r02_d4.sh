# speculative next-round IDs only where few fronts run (HSSMF_SPEC_PEERS), tests, launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_spec.py tests/test_gpu_hss.py tests/test_gpu_mf.py -x -q > gpurun_out/d4_tests.txt 2>&1; echo "tests rc=$?"
tail -n 3 gpurun_out/d4_tests.txt
run() { tag=$1; shift; env "$@" timeout 900 python bench.py --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/d4_bench_$tag.json 2> gpurun_out/d4_bench_$tag.err; echo "bench $tag rc=$?"; python -c "
import json
d=json.loads(open('gpurun_out/d4_bench_$tag.json').read().strip().splitlines()[-1]); print('$tag', d['value'], d['e2e']['value'], d['relres'])"; }
run base A=1
run peers4 HSSMF_SPEC_PEERS=4
run peers4_r1500 HSSMF_SPEC_PEERS=4 HSSMF_SPEC_ID_ROWS=1500
run peers2 HSSMF_SPEC_PEERS=2
run peers8 HSSMF_SPEC_PEERS=8
CMD="python tools/gpu_fronts.py c5 --out gpurun_out/ncu_plain.npz"
timeout 2700 ncu --metrics gpu__time_duration.sum --clock-control none -c 60000 --csv \
    --log-file /tmp/r02_launches_c5.csv $CMD > gpurun_out/ncu_list.log 2>&1; echo "list rc=$?"
ls -la /tmp/r02_launches_c5.csv; head -c 600 /tmp/r02_launches_c5.csv
python - <<'P' > gpurun_out/r02_launches_c5_summary.txt 2>&1
import csv, collections, re
t = collections.defaultdict(lambda: [0, 0.0])
n = 0
rows = []
with open('/tmp/r02_launches_c5.csv', newline='') as f:
    for r in csv.reader(f):
        rows.append(r)
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
hdr = rows[hi]
ki, vi, ui = hdr.index('Kernel Name'), hdr.index('Metric Value'), hdr.index('Metric Unit')
for r in rows[hi + 1:]:
    if len(r) <= max(ki, vi, ui): continue
    try: v = float(r[vi].replace(',', ''))
    except ValueError: continue
    u = r[ui]
    v *= {'ns': 1e-3, 'us': 1.0, 'usecond': 1.0, 'nsecond': 1e-3, 'msecond': 1e3, 'ms': 1e3, 'second': 1e6, 's': 1e6}.get(u, 1.0)
    name = re.sub(r'\(.*', '', r[ki])
    t[name][0] += 1; t[name][1] += v; n += 1
tot = sum(v[1] for v in t.values())
print("first %d launches of one c5 factorization + solve (ncu --metrics gpu__time_duration.sum --clock-control none), total %.1f ms" % (n, tot / 1e3))
for k, v in sorted(t.items(), key=lambda kv: -kv[1][1]):
    print("%-60s %7d launches %10.1f ms %5.1f%% %8.1f us/launch" % (k[:60], v[0], v[1] / 1e3, 100 * v[1] / tot, v[1] / v[0]))
P
head -n 20000 /tmp/r02_launches_c5.csv | gzip > gpurun_out/r02_launches_c5_first20000.csv.gz
du -sh gpurun_out
