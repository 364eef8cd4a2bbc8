mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "real_data" > gpurun_out/pytest_gpu25a.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu25a.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu25.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu25.log
