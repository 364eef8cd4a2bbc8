mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "dense" > gpurun_out/pytest_gpu35a.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu35a.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu35.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu35.log
