# ncu --set full capture of the CQ T-pass on C5 (after a clean run without ncu).
mkdir -p gpurun_out
timeout 300 python bench.py --config C5 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/pre_cq.json 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tpass_kernel -s 2 -c 1 -o gpurun_out/prof_cq_tpass -f python bench.py --config C5 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_cq.log 2>&1
