mkdir -p gpurun_out
for r in 1 2; do
  PINT_LIB=ab/libpint_head.so timeout 300 python bench.py --config C5 --no-cpu --no-e2e > gpurun_out/ab52_head_$r.json 2>> gpurun_out/ab52.err
  timeout 300 python bench.py --config C5 --no-cpu --no-e2e > gpurun_out/ab52_new_$r.json 2>> gpurun_out/ab52.err
done
