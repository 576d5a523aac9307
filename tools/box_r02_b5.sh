# Gram panel / SYRK microbenchmarks: per-step latency and segment cycles
mkdir -p gpurun_out
for cl in 16 8 4; do
  HSSMF_GRAM_MAXCL=$cl HSSMF_GRAM_TPROBE=1 timeout 300 python tools/gram_bench.py > gpurun_out/b5_gram_cl$cl.json 2> gpurun_out/b5_gram_cl$cl.err
done
HSSMF_GRAM_SYRK=persist timeout 300 python tools/gram_bench.py > gpurun_out/b5_gram_persist.json 2>&1
timeout 300 python tools/gemm_shapes.py > gpurun_out/b5_gemm_shapes.json 2> gpurun_out/b5_gemm_shapes.err
