# final-build evidence: c5 fronts vs the reference run, launch list, --set full captures
mkdir -p gpurun_out
CMD="python tools/gpu_fronts.py c5 --out gpurun_out/d13_c5.npz"
$CMD > gpurun_out/d13_c5.log 2>&1; echo "plain rc=$?"; tail -n 1 gpurun_out/d13_c5.log
python tools/compare_fronts.py gpurun_out/d13_c5.npz tests/golden/ref_c5.npz > gpurun_out/d13_c5_vs_reference.txt 2>&1; cat gpurun_out/d13_c5_vs_reference.txt
CMD="python tools/gpu_fronts.py c5 --out gpurun_out/ncu_plain.npz"
for spec in "gemm_tma:-s 20 -c 2" "gemm_param_kernel:-s 3000 -c 2" "gram_syrk_dmma:-s 20000 -c 1" "gram_panel2:-s 20000 -c 1" "tri_inv:-s 50 -c 1"; do
  k=${spec%%:*}; a=${spec#*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k $a \
    -o /tmp/r02f_$k -f $CMD > gpurun_out/ncu_$k.log 2>&1; echo "$k rc=$?"
  ncu -i /tmp/r02f_$k.ncu-rep --page details > gpurun_out/r02_final_${k}_details.txt 2>&1
  ncu -i /tmp/r02f_$k.ncu-rep --page raw --csv > gpurun_out/r02_final_${k}_raw.csv 2>&1
  rm -f /tmp/r02f_$k.ncu-rep
done
timeout 2700 ncu --metrics gpu__time_duration.sum --clock-control none -c 60000 --csv \
    --log-file /tmp/r02f_launches_c5.csv $CMD > gpurun_out/ncu_list.log 2>&1; echo "list rc=$?"
python - <<'P' > gpurun_out/r02_final_launches_c5_summary.txt 2>&1
import csv, collections, re
t = collections.defaultdict(lambda: [0, 0.0])
n = 0
rows = []
with open('/tmp/r02f_launches_c5.csv', newline='') as f:
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
head -n 20000 /tmp/r02f_launches_c5.csv | gzip > gpurun_out/r02_final_launches_c5_first20000.csv.gz
du -sh gpurun_out
