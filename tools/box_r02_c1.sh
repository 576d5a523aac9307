# re-entry check: full GPU suite, smoke, default bench
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/c1_gpu_tests.txt 2>&1; echo "tests rc=$?"
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c1_smoke.txt 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/c1_bench.json 2> gpurun_out/c1_bench.err; echo "bench rc=$?"
tail -c 600 gpurun_out/c1_gpu_tests.txt
