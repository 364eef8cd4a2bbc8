mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu22.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu22.log
timeout 300 python bench.py --no-cpu --no-e2e --steps 10 > gpurun_out/bench22.json 2> gpurun_out/bench22.err
