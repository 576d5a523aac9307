# round-2 GPU check 3: K-routed TMA GEMM, Gram tail check at C5 / C3 / C4 parity
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k gemm > gpurun_out/b3_gemm_tests.txt 2>&1
HSSMF_DEBUG=1 timeout 900 python tools/gpu_fronts.py c5 --out gpurun_out/b3_gpu_c5.npz > gpurun_out/b3_debug.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_hss.py -q -k "baseline_config or config5 or p3d_with" > gpurun_out/b3_parity.txt 2>&1
timeout 300 python tools/gemm_shapes.py > gpurun_out/b3_gemm_shapes.json 2> gpurun_out/b3_gemm_shapes.err
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/b3_bench.json 2> gpurun_out/b3_bench.err
