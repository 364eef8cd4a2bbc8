mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -q -x -k "unread and fused or c1_parity or c2_sweep" > gpurun_out/pytest_gpu7.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu7.log
for d in 0 1 2 4 6 7; do
  PINT_FUSED_DBG=$d timeout 300 python bench.py --no-cpu --no-e2e --steps 5 > gpurun_out/bench7_dbg$d.json 2> gpurun_out/bench7_dbg$d.err
done
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:wr_fused_kernel -s 3 -c 1 -o gpurun_out/prof_fused_v4 -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --mx 127 > gpurun_out/ncu_full7.log 2>&1
