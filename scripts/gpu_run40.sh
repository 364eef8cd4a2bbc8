mkdir -p gpurun_out
for r in 1 2; do
  PINT_LIB=ab/libpint_base.so timeout 300 python bench.py --no-cpu --no-e2e > gpurun_out/ab40_base_$r.json 2>> gpurun_out/ab40.err
  timeout 300 python bench.py --no-cpu --no-e2e > gpurun_out/ab40_new_$r.json 2>> gpurun_out/ab40.err
done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/pytest_gpu40.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu40.log
