# C5 determinism (same build twice), one-ulp input perturbations, pivot dump
mkdir -p gpurun_out
timeout 900 python tools/gpu_fronts.py c5 --out gpurun_out/c3_plain.npz --repeat 2 > gpurun_out/c3_plain.log 2>&1; echo "plain rc=$?"
for sd in 1 2 3; do
  timeout 600 python tools/gpu_fronts.py c5 --perturb $sd --out gpurun_out/c3_pert$sd.npz > gpurun_out/c3_pert$sd.log 2>&1; echo "pert $sd rc=$?"
done
HSSMF_DUMP_PIVOTS=gpurun_out/c3_piv.bin timeout 900 python tools/gpu_fronts.py c5 --out gpurun_out/c3_dump.npz > gpurun_out/c3_dump.log 2>&1; echo "dump rc=$?"
ls -la gpurun_out/c3_piv.bin
cat gpurun_out/c3_*.log
