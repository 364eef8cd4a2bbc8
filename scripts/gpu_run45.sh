mkdir -p gpurun_out
for r in 1 2; do
  PINT_LIB=ab/libpint_1f7.so timeout 300 python bench.py --config C5 --no-cpu --no-e2e > gpurun_out/ab45_old_$r.json 2>> gpurun_out/ab45.err
  timeout 300 python bench.py --config C5 --no-cpu --no-e2e > gpurun_out/ab45_new_$r.json 2>> gpurun_out/ab45.err
done
