mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -q -x -k "unread and fused" > gpurun_out/pytest_gpu5a.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu5a.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu5.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu5.log
timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/bench5.json 2> gpurun_out/bench5.err
PINT_FUSED_V1=1 timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/bench5_v1.json 2> gpurun_out/bench5_v1.err
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:wr_fused2_kernel -s 3 -c 1 -o gpurun_out/prof_fused_v2 -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --mx 127 > gpurun_out/ncu_full5.log 2>&1
