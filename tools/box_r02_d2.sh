# session 3 baseline (outputs kept small: gpurun_out is limited to 64 MiB)
mkdir -p gpurun_out
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/d2_bench.json 2> gpurun_out/d2_bench.err; echo "bench rc=$?"
HSSMF_DUMP_PIVOTS=/tmp/d2_piv.bin timeout 900 python tools/gpu_fronts.py c5 --out gpurun_out/d2_dump.npz > gpurun_out/d2_dump.log 2>&1; echo "dump rc=$?"
python tools/pivot_replay.py /tmp/d2_piv.bin --block 48 > gpurun_out/d2_replay48.txt 2>&1
python tools/pivot_replay.py /tmp/d2_piv.bin --block 16 > gpurun_out/d2_replay16.txt 2>&1
python tools/pivot_rounds.py /tmp/d2_piv.bin --top 80 > gpurun_out/d2_rounds.txt 2>&1
gzip -c /tmp/d2_piv.bin > gpurun_out/d2_piv.bin.gz; rm -f /tmp/d2_piv.bin
HSSMF_DEBUG=1 timeout 900 python tools/gpu_fronts.py c5 --out gpurun_out/d2_dbg.npz > gpurun_out/d2_dbg.log 2>&1; echo "dbg rc=$?"
HSSMF_DEBUG=1 HSSMF_HSS_STREAMS=1 timeout 900 python tools/gpu_fronts.py c5 --out gpurun_out/d2_dbg1.npz > gpurun_out/d2_dbg1.log 2>&1; echo "dbg1 rc=$?"
CMD="python tools/gpu_fronts.py c5 --out gpurun_out/ncu_plain.npz"
for spec in "gemm_tma:-s 20 -c 2" "gemm_param_kernel:-s 3000 -c 2" "extend_add:-s 14 -c 4" "gram_syrk_dmma:-s 30000 -c 1" "gram_panel2:-s 30000 -c 1"; do
  k=${spec%%:*}; a=${spec#*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k $a \
    -o /tmp/r02_$k -f $CMD > gpurun_out/ncu_$k.log 2>&1; echo "$k rc=$?"
  ncu -i /tmp/r02_$k.ncu-rep --page details > gpurun_out/r02_${k}_details.txt 2>&1
  ncu -i /tmp/r02_$k.ncu-rep --page raw --csv > gpurun_out/r02_${k}_raw.csv 2>&1
  rm -f /tmp/r02_$k.ncu-rep
done
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 90000 --csv \
    --log-file /tmp/r02_launches_c5.csv $CMD > gpurun_out/ncu_list.log 2>&1; echo "list rc=$?"
python - <<'P' > gpurun_out/r02_launches_c5_summary.txt 2>&1
import csv, collections, re
t = collections.defaultdict(lambda: [0, 0.0])
n = 0
with open('/tmp/r02_launches_c5.csv') as f:
    rows = [r for r in csv.reader(l for l in f if not l.startswith('=='))]
hdr = rows[0]
ki, vi, ui = hdr.index('Kernel Name'), hdr.index('Metric Value'), hdr.index('Metric Unit')
for r in rows[1:]:
    if len(r) <= vi: continue
    v = float(r[vi].replace(',', ''))
    u = r[ui]
    v *= {'ns': 1e-3, 'us': 1.0, 'usecond': 1.0, 'nsecond': 1e-3, 'msecond': 1e3, 'ms': 1e3}.get(u, 1.0)
    name = re.sub(r'\(.*', '', r[ki])
    t[name][0] += 1; t[name][1] += v; n += 1
tot = sum(v[1] for v in t.values())
print("first %d launches of one c5 factorization + solve (ncu --metrics gpu__time_duration.sum --clock-control none), total %.1f ms" % (n, tot / 1e3))
for k, v in sorted(t.items(), key=lambda kv: -kv[1][1]):
    print("%-60s %7d launches %10.1f ms %5.1f%% %8.1f us/launch" % (k[:60], v[0], v[1] / 1e3, 100 * v[1] / tot, v[1] / v[0]))
P
head -c 3000000 /tmp/r02_launches_c5.csv | gzip > gpurun_out/r02_launches_c5_head.csv.gz
du -sh gpurun_out; ls -la gpurun_out
