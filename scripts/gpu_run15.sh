mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu15.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu15.log
timeout 600 python bench.py --dst-per-iter --no-cpu --no-e2e --steps 5 > gpurun_out/bench15_dstiter.json 2> gpurun_out/bench15_dstiter.err
