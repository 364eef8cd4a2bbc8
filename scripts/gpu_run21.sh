mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu21.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu21.log
timeout 300 python bench.py --no-cpu --no-e2e --steps 10 > gpurun_out/bench21.json 2> gpurun_out/bench21.err
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:wr_fused_kernel -s 3 -c 1 -o gpurun_out/prof_fused_v9 -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --mx 127 > gpurun_out/ncu_full21.log 2>&1
