mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "unread or c1_parity or pruned or state_errors" > gpurun_out/pytest_gpu3a.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu3a.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu3.log
timeout 600 python bench.py --no-cpu > gpurun_out/bench3.json 2> gpurun_out/bench3.err
