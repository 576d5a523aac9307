# NB2 = 48 Gram panels (fixed push), batched HSS-front assembly: microbench, tests, bench
mkdir -p gpurun_out
HSSMF_GRAM_TPROBE=1 timeout 120 python tools/gram_bench.py > gpurun_out/b7_gram.json 2> gpurun_out/b7_gram.err || { echo "gram bench failed"; exit 1; }
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_spec.py -x -q > gpurun_out/b7_kernel_tests.txt 2>&1 || { echo "kernel tests failed"; exit 1; }
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/b7_bench.json 2> gpurun_out/b7_bench.err
HSSMF_HSS_STREAMS=8 timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/b7_bench_w8.json 2> gpurun_out/b7_bench_w8.err
timeout 1500 python -m pytest tests/test_gpu_hss.py -q -k "baseline_config or config5 or p3d_with" > gpurun_out/b7_parity.txt 2>&1
