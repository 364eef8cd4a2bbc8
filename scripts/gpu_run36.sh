mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -q -x -k "divergence" > gpurun_out/pytest_gpu36.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu36.log
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:tpass_kernel -s 2 -c 1 -o gpurun_out/prof_cq_v2 -f python bench.py --config C5 --steps 1 --warmup 2 --no-e2e --no-cpu > gpurun_out/ncu_cq2.log 2>&1
