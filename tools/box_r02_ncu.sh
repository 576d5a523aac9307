# ncu evidence for round 2 (run only after the same command exited 0 plainly):
# launch list of one c5 factorization + solve, then --set full on the judged kernels
mkdir -p gpurun_out
CMD="python tools/gpu_fronts.py c5 --out gpurun_out/ncu_plain.npz"
$CMD > gpurun_out/ncu_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 330000 --csv \
    --log-file gpurun_out/r02_launches_c5.csv $CMD > gpurun_out/ncu_list.log 2>&1
for spec in "gemm_tma:-s 20 -c 2" "gemm_param_kernel:-s 3000 -c 2" "extend_add:-s 14 -c 6" "gram_syrk_dmma:-s 30000 -c 1" "gram_panel2:-s 30000 -c 1"; do
  k=${spec%%:*}; a=${spec#*:}
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$k $a \
    -o gpurun_out/r02_$k $CMD > gpurun_out/ncu_$k.log 2>&1
done
