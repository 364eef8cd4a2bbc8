mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu6.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu6.log
timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/bench6.json 2> gpurun_out/bench6.err
PINT_FUSED_LANES=64 timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/bench6_l64.json 2> gpurun_out/bench6_l64.err
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:wr_fused_kernel -s 3 -c 1 -o gpurun_out/prof_fused_v3 -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --mx 127 > gpurun_out/ncu_full6.log 2>&1
