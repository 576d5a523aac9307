# round-2 GPU check: new GEMM paths, HSS matvec/extract KATs, bench, C5 debug, full GPU suite
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/b2_smi.txt 2>&1
nproc > gpurun_out/b2_host.txt; free -g >> gpurun_out/b2_host.txt
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k gemm > gpurun_out/b2_gemm_tests.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_hss.py -q -k "matvec or extract or full_size" > gpurun_out/b2_hss_tests.txt 2>&1
timeout 300 python tools/gemm_shapes.py > gpurun_out/b2_gemm_shapes.json 2> gpurun_out/b2_gemm_shapes.err
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/b2_bench.json 2> gpurun_out/b2_bench.err
HSSMF_DEBUG=1 timeout 600 python tools/gpu_fronts.py c5 --out gpurun_out/b2_gpu_c5.npz > gpurun_out/b2_debug.txt 2>&1
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/b2_gpu_tests.txt 2>&1
