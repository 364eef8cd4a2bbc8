mkdir -p gpurun_out
timeout 300 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --mx 127 > gpurun_out/pre41.json 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:wr_fused_kernel -s 3 -c 1 -o gpurun_out/prof_fused_v10 -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --mx 127 > gpurun_out/ncu_full41.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches41.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch41.log 2>&1
