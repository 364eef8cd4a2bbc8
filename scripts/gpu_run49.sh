mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "fem or modal or smoke or c1_parity" > gpurun_out/pytest49.log 2>&1; echo "rc=$?" >> gpurun_out/pytest49.log
timeout 300 python bench.py --modal --no-cpu --no-e2e > gpurun_out/b49_modal.json 2>> gpurun_out/b49.err
