set -x
python -m pytest tests -m gpu -x -q -k "cq or c5 or C5 or full or two_processes or random_complex or slabs or residual or dense or modal or newton" -m "gpu and not slow" > gpurun_out/t2.log 2>&1
tail -5 gpurun_out/t2.log
python bench.py --config C5 --steps 10 --warmup 3 --no-cpu > gpurun_out/b2_c5.json 2> gpurun_out/b2_c5.err
python bench.py --config C3 --gpus 2 --steps 5 --warmup 3 --no-cpu > gpurun_out/b2_c3_g2.json 2> gpurun_out/b2_c3_g2.err
timeout 600 ncu --set full --import-source on -k regex:tpass_cq_fused -c 1 -o gpurun_out/prof_cqf_v1 python bench.py --config C5 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_cqf_v1.log 2>&1
tail -3 gpurun_out/ncu_cqf_v1.log
