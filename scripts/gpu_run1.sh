set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
for v in PINT_SPASS_STAGED PINT_SPASS_DIRECT PINT_NO_PREFETCH; do
  env $v=1 timeout 300 python bench.py --no-e2e --no-cpu > gpurun_out/bench_$v.json 2> gpurun_out/bench_$v.err
done
PINT_ALLOC=vmm_comp timeout 300 python bench.py --no-e2e --no-cpu > gpurun_out/bench_vmmcomp.json 2> gpurun_out/bench_vmmcomp.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
