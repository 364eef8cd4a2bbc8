mkdir -p gpurun_out
for r in 1 2; do
  PINT_LIB=ab/libpint_cqminb1.so timeout 300 python bench.py --config C5 --no-cpu --no-e2e > gpurun_out/ab47_minb1_$r.json 2>> gpurun_out/ab47.err
  timeout 300 python bench.py --config C5 --no-cpu --no-e2e > gpurun_out/ab47_cur_$r.json 2>> gpurun_out/ab47.err
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tpass_kernel -s 2 -c 1 -o gpurun_out/prof_cq_tpass_v1 -f python bench.py --config C5 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu47.log 2>&1
