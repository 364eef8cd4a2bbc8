mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu32.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu32.log
timeout 600 python bench.py --config C3 --no-cpu > gpurun_out/bench32_C3.json 2> gpurun_out/bench32_C3.err
timeout 600 python bench.py --no-cpu > gpurun_out/bench32.json 2> gpurun_out/bench32.err
