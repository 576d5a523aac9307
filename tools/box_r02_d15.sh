mkdir -p gpurun_out
HSSMF_DEBUG_AN=1 timeout 600 python tools/gpu_fronts.py c5 --out gpurun_out/d15_c5.npz > gpurun_out/d15_c5.log 2>&1; grep analyze gpurun_out/d15_c5.log; tail -n 1 gpurun_out/d15_c5.log
