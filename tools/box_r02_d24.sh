mkdir -p gpurun_out
HSSMF_DEBUG=1 timeout 900 python tools/gpu_fronts.py c5 --out gpurun_out/d24_dbg.npz > gpurun_out/d24_dbg.log 2>&1; echo "rc=$?"; grep "level:" gpurun_out/d24_dbg.log; grep -A5 "level: 4 HSS fronts" gpurun_out/d24_dbg.log | cut -c1-250; tail -n 1 gpurun_out/d24_dbg.log
