mkdir -p gpurun_out
for r in 1 2; do
  PINT_LIB=ab/libpint_1f7.so timeout 300 python bench.py --config C5 --no-cpu --no-e2e > gpurun_out/ab46_old_$r.json 2>> gpurun_out/ab46.err
  timeout 300 python bench.py --config C5 --no-cpu --no-e2e > gpurun_out/ab46_new_$r.json 2>> gpurun_out/ab46.err
done
PINT_LIB=ab/libpint_1f7.so timeout 300 python bench.py --path stream --no-cpu --no-e2e > gpurun_out/ab46_old_stream.json 2>> gpurun_out/ab46.err
timeout 300 python bench.py --path stream --no-cpu --no-e2e > gpurun_out/ab46_new_stream.json 2>> gpurun_out/ab46.err
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "dense or newton or c5 or random_complex or unread" > gpurun_out/pytest46.log 2>&1; echo "rc=$?" >> gpurun_out/pytest46.log
