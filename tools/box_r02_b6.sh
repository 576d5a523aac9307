# NB2 = 48 Gram panels: per-step latency, parity, bench
mkdir -p gpurun_out
HSSMF_GRAM_TPROBE=1 timeout 300 python tools/gram_bench.py > gpurun_out/b6_gram.json 2> gpurun_out/b6_gram.err
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_spec.py -x -q > gpurun_out/b6_kernel_tests.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_hss.py -q -k "baseline_config or config5 or p3d_with" > gpurun_out/b6_parity.txt 2>&1
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/b6_bench.json 2> gpurun_out/b6_bench.err
