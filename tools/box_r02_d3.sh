# round schedule (failing IDs extrapolated, downward checks, joined rounds): parity and speed
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_spec.py -x -q > gpurun_out/d3_spec_tests.txt 2>&1; echo "spec tests rc=$?"
HSSMF_DEBUG_ROUNDS=1 timeout 600 python tools/gpu_fronts.py c3 --out gpurun_out/d3_c3.npz > gpurun_out/d3_c3.log 2>&1; echo "c3 rc=$?"
HSSMF_DEBUG_ROUNDS=1 timeout 900 python tools/gpu_fronts.py c5 --out gpurun_out/d3_c5.npz > gpurun_out/d3_c5.log 2>&1; echo "c5 rc=$?"
timeout 900 python bench.py --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/d3_bench.json 2> gpurun_out/d3_bench.err; echo "bench rc=$?"
HSSMF_EXACT_ROUNDS=1 timeout 900 python bench.py --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/d3_bench_exact.json 2> gpurun_out/d3_bench_exact.err; echo "bench exact rc=$?"
timeout 1500 python -m pytest tests/test_gpu_hss.py tests/test_gpu_mf.py -x -q > gpurun_out/d3_tests.txt 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/d3_spec_tests.txt gpurun_out/d3_tests.txt
du -sh gpurun_out
