mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu8.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu8.log
for d in 0 8 1 6; do
  PINT_FUSED_DBG=$d timeout 300 python bench.py --no-cpu --no-e2e --steps 5 > gpurun_out/bench8_dbg$d.json 2> gpurun_out/bench8_dbg$d.err
done
