mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -k graph_replay > gpurun_out/pytest_graph38.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_graph38.log
for c in C1 C2; do
  timeout 300 python bench.py --config $c --no-cpu > gpurun_out/bench38_$c.json 2> gpurun_out/bench38_$c.err
  PINT_NO_GRAPH=1 timeout 300 python bench.py --config $c --no-cpu > gpurun_out/bench38_${c}_eager.json 2>> gpurun_out/bench38_$c.err
done
timeout 600 python bench.py > gpurun_out/bench38_C4.json 2> gpurun_out/bench38_C4.err
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu38.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu38.log
