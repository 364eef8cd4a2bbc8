# CQ T-pass iteration: parity subset, C5 bench, ncu of the one-kernel T-pass
python -m pytest tests -x -q -m "gpu and not slow" -k "cq or c5 or C5 or full or two_processes or random_complex or slabs or residual or modal" > gpurun_out/t3.log 2>&1
tail -3 gpurun_out/t3.log
python bench.py --config C5 --steps 10 --warmup 3 --no-cpu > gpurun_out/b3_c5.json 2> gpurun_out/b3_c5.err
timeout 600 ncu --set full --import-source on -k regex:tpass_cq_fused -c 1 -o gpurun_out/prof_cqf_v2 python bench.py --config C5 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_cqf_v2.log 2>&1
tail -2 gpurun_out/ncu_cqf_v2.log
