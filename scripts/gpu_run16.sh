mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -q -x -k "c1_parity or unread or c2_sweep" > gpurun_out/pytest_gpu16a.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu16a.log
timeout 300 python bench.py --no-cpu --no-e2e --steps 10 > gpurun_out/bench16_tmem.json 2> gpurun_out/bench16_tmem.err
PINT_FUSED_TMEM=0 timeout 300 python bench.py --no-cpu --no-e2e --steps 10 > gpurun_out/bench16_smem.json 2> gpurun_out/bench16_smem.err
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu16.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu16.log
