mkdir -p gpurun_out
timeout 600 python bench.py --real --no-cpu > gpurun_out/bench26_real.json 2> gpurun_out/bench26_real.err
timeout 600 python bench.py --real --config C3 --no-cpu > gpurun_out/bench26_real_C3.json 2> gpurun_out/bench26_real_C3.err
