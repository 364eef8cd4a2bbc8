mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu37.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu37.log
for c in C1 C2; do timeout 600 python bench.py --config $c --no-cpu > gpurun_out/bench37_$c.json 2> gpurun_out/bench37_$c.err; done
