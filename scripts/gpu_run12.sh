mkdir -p gpurun_out
PINT_FUSED_LANES=64 timeout 300 python bench.py --no-cpu --no-e2e --steps 5 > gpurun_out/bench12_l64.json 2> gpurun_out/bench12_l64.err
PINT_LIB=$PWD/paper_2007_13125_b200/libpint_cq2.so timeout 300 python bench.py --config C5 --no-cpu --no-e2e --steps 5 > gpurun_out/bench12_c5_cq2.json 2> gpurun_out/bench12_c5_cq2.err
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:tpass_kernel -s 2 -c 1 -o gpurun_out/prof_cq_v1 -f python bench.py --config C5 --steps 1 --warmup 2 --no-e2e --no-cpu > gpurun_out/ncu_cq.log 2>&1
