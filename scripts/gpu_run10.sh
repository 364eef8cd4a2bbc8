mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu10.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu10.log
for d in 0 1 6 7; do
  PINT_FUSED_DBG=$d timeout 300 python bench.py --no-cpu --no-e2e --steps 5 > gpurun_out/bench10_dbg$d.json 2> gpurun_out/bench10_dbg$d.err
done
PINT_FUSED_KERNEL=r8 timeout 300 python bench.py --no-cpu --no-e2e --steps 5 > gpurun_out/bench10_r8.json 2> gpurun_out/bench10_r8.err
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:wr_fused_ws_kernel -s 3 -c 1 -o gpurun_out/prof_fused_ws1 -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --mx 127 > gpurun_out/ncu_full10.log 2>&1
