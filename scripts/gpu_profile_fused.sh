# ncu --set full capture of the fused kernel on a 127-x-mode C4 slab (after a clean run without ncu).
mkdir -p gpurun_out
timeout 300 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --mx 127 > gpurun_out/pre_fused.json 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:wr_fused_kernel -s 3 -c 1 -o gpurun_out/prof_fused -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --mx 127 > gpurun_out/ncu_fused.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_fused.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch_fused.log 2>&1
