mkdir -p gpurun_out
HSSMF_DEBUG=1 timeout 900 python tools/gpu_fronts.py c5 --repeat 3 --out gpurun_out/d25_dbg.npz > gpurun_out/d25_dbg.log 2>&1; echo "rc=$?"; grep "level:" gpurun_out/d25_dbg.log | tail -n 8; grep "^c5" gpurun_out/d25_dbg.log
