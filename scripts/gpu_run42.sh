mkdir -p gpurun_out
for r in 1 2; do
  for v in cur ns2 ns8; do
    if [ $v = cur ]; then L=""; else L="PINT_LIB=ab/libpint_$v.so"; fi
    env $L timeout 300 python bench.py --no-cpu --no-e2e > gpurun_out/ab42_${v}_$r.json 2>> gpurun_out/ab42.err
  done
done
