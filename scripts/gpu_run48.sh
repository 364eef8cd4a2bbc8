mkdir -p gpurun_out
for r in 1 2; do
  PINT_LIB=ab/libpint_base.so timeout 300 python bench.py --config C5 --no-cpu --no-e2e > gpurun_out/ab48_base_$r.json 2>> gpurun_out/ab48.err
  timeout 300 python bench.py --config C5 --no-cpu --no-e2e > gpurun_out/ab48_new_$r.json 2>> gpurun_out/ab48.err
done
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "c5 or random_complex or dense or newton or stream" > gpurun_out/pytest48.log 2>&1; echo "rc=$?" >> gpurun_out/pytest48.log
