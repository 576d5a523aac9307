# session 3 baseline: bench line, pivot dump for the replay study, launch list + --set full captures
mkdir -p gpurun_out
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/d1_bench.json 2> gpurun_out/d1_bench.err; echo "bench rc=$?"
HSSMF_DUMP_PIVOTS=gpurun_out/d1_piv.bin timeout 900 python tools/gpu_fronts.py c5 --out gpurun_out/d1_dump.npz > gpurun_out/d1_dump.log 2>&1; echo "dump rc=$?"
ls -la gpurun_out/d1_piv.bin
python tools/pivot_replay.py gpurun_out/d1_piv.bin --block 48 > gpurun_out/d1_replay48.txt 2>&1
python tools/pivot_replay.py gpurun_out/d1_piv.bin --block 16 > gpurun_out/d1_replay16.txt 2>&1
gzip -f gpurun_out/d1_piv.bin
CMD="python tools/gpu_fronts.py c5 --out gpurun_out/ncu_plain.npz"
timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none -c 260000 --csv \
    --log-file gpurun_out/r02_launches_c5.csv $CMD > gpurun_out/ncu_list.log 2>&1; echo "list rc=$?"
for spec in "gemm_tma:-s 20 -c 2" "gemm_param_kernel:-s 3000 -c 2" "extend_add:-s 14 -c 6" "gram_syrk_dmma:-s 30000 -c 1" "gram_panel2:-s 30000 -c 1"; do
  k=${spec%%:*}; a=${spec#*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k $a \
    -o gpurun_out/r02_$k $CMD > gpurun_out/ncu_$k.log 2>&1; echo "$k rc=$?"
done
ls -la gpurun_out
