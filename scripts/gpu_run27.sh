mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "modal" > gpurun_out/pytest_gpu27a.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu27a.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu27.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu27.log
