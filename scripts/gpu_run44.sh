mkdir -p gpurun_out
for c in C4 C1 C2 C3 C5; do timeout 300 python bench.py --config $c --no-cpu > gpurun_out/b44_$c.json 2>> gpurun_out/b44.err; done
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest44.log 2>&1; echo "rc=$?" >> gpurun_out/pytest44.log
