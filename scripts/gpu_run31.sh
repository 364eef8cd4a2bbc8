mkdir -p gpurun_out
PINT_FUSED_LANES=64 timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/bench31_l64.json 2> gpurun_out/bench31_l64.err
timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/bench31_l32.json 2> gpurun_out/bench31_l32.err
