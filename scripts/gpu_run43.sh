mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "graph_replay or timing or c1_parity" > gpurun_out/pytest43.log 2>&1; echo "rc=$?" >> gpurun_out/pytest43.log
for c in C4 C1 C2 C3; do timeout 300 python bench.py --config $c --no-cpu > gpurun_out/b43_$c.json 2>> gpurun_out/b43.err; done
