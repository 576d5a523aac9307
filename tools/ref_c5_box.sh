#!/bin/bash
# BASELINE config 5 (P3D 128^3) on one GPU box: the product's per-front ranks for the
# default route and the two shortcut-free variants, then the reference (oracle/_ref) on
# all host cores. Writes gpurun_out/{gpu_c5*.npz,ref_c5.npz,...}. Test infrastructure only.
set -u
mkdir -p gpurun_out
{ nproc; free -g; lscpu | head -20; } > gpurun_out/ref_c5_host.txt 2>&1
if [ -z "${SKIP_GPU:-}" ]; then
  timeout 900 python tools/gpu_fronts.py c5 --out gpurun_out/gpu_c5.npz >> gpurun_out/gpu_c5.log 2>&1
  HSSMF_NO_SYM=1 timeout 900 python tools/gpu_fronts.py c5 --out gpurun_out/gpu_c5_nosym.npz >> gpurun_out/gpu_c5.log 2>&1
  HSSMF_ID_ALGO=householder timeout 1500 python tools/gpu_fronts.py c5 --out gpurun_out/gpu_c5_hh.npz >> gpurun_out/gpu_c5.log 2>&1
fi
timeout ${REF_TIMEOUT:-6000} python tests/golden/make_golden.py ${REF_CFG:-c5} \
  --out-dir gpurun_out > gpurun_out/ref_c5.log 2> gpurun_out/ref_c5.err
echo "rc=$?" >> gpurun_out/ref_c5.log
