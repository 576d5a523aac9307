# reference arm and its scaling validation on the GPU-box host (CPU work)
mkdir -p gpurun_out
timeout 1500 python tools/validate_ref_scaling.py c3 c5_96 --budget 60 --steps 3 > gpurun_out/val_scaling.json 2> gpurun_out/val_scaling.err
( time timeout 900 python bench.py --impl reference --steps 20 --warmup 5 ) > gpurun_out/val_refarm.json 2> gpurun_out/val_refarm.err
