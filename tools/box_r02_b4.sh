# round-2 GPU check 4: persistent Gram SYRK, small-tile rule, parity + bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_spec.py -x -q > gpurun_out/b4_kernel_tests.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_hss.py -q -k "baseline_config or config5 or p3d_with" > gpurun_out/b4_parity.txt 2>&1
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/b4_bench.json 2> gpurun_out/b4_bench.err
HSSMF_DEBUG=1 timeout 900 python tools/gpu_fronts.py c5 --out gpurun_out/b4_gpu_c5.npz > gpurun_out/b4_debug.txt 2>&1
