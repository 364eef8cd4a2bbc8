mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "graph_replay or c1_parity or c2_sweep or unread or slabs" > gpurun_out/pytest_graph39.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_graph39.log
for c in C1 C2; do
  timeout 300 python bench.py --config $c --no-cpu > gpurun_out/bench39_$c.json 2> gpurun_out/bench39_$c.err
done
timeout 600 python bench.py > gpurun_out/bench39_C4.json 2> gpurun_out/bench39_C4.err
