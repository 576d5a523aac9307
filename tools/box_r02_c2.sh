# full GPU suite after the test fix, then compute-sanitizer memcheck on the small cases
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/c2_gpu_tests.txt 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/c2_gpu_tests.txt
timeout 1500 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize_small.py > gpurun_out/c2_memcheck.txt 2>&1; echo "memcheck rc=$?"
tail -15 gpurun_out/c2_memcheck.txt
