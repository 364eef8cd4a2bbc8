mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "newton" -s > gpurun_out/pytest_gpu24a.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu24a.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu24.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu24.log
