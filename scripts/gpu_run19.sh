mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -q -x -k "c1_parity or unread or c2_sweep" > gpurun_out/pytest_gpu19a.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu19a.log
timeout 300 python bench.py --no-cpu --no-e2e --steps 10 > gpurun_out/bench19_r4.json 2> gpurun_out/bench19_r4.err
PINT_FUSED_KERNEL=r8 timeout 300 python bench.py --no-cpu --no-e2e --steps 10 > gpurun_out/bench19_r8.json 2> gpurun_out/bench19_r8.err
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu19.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu19.log
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:wr_fused4_kernel -s 3 -c 1 -o gpurun_out/prof_fused4_v1 -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --mx 127 > gpurun_out/ncu_full19.log 2>&1
