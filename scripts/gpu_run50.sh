mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "fem or modal" -s > gpurun_out/pytest50.log 2>&1; echo "rc=$?" >> gpurun_out/pytest50.log
timeout 300 python bench.py --config C5 --modal --no-cpu --no-e2e > gpurun_out/b50_c5modal.json 2>> gpurun_out/b50.err
