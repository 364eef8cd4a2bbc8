mkdir -p gpurun_out
for v in ns2 ns8; do
  PINT_LIB=$PWD/paper_2007_13125_b200/libpint_$v.so timeout 300 python bench.py --no-cpu --no-e2e --steps 5 > gpurun_out/bench13_$v.json 2> gpurun_out/bench13_$v.err
done
timeout 300 python bench.py --no-cpu --no-e2e --steps 5 > gpurun_out/bench13_ns4.json 2> gpurun_out/bench13_ns4.err
for c in C3 C5; do PINT_LIB=$PWD/paper_2007_13125_b200/libpint_cq2.so timeout 300 python bench.py --config $c --path stream --no-cpu --no-e2e --steps 5 > gpurun_out/bench13_${c}_cq2.json 2> gpurun_out/bench13_${c}_cq2.err; done
