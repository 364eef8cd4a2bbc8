# CQ T-pass A/B: default (2 CTAs/SM) vs variant lib (3 CTAs/SM); parity subset first
python -m pytest tests -x -q -m "gpu and not slow" -k "cq or c5 or C5 or full or random_complex or residual or modal or slabs" > gpurun_out/t5.log 2>&1
tail -2 gpurun_out/t5.log
for r in 1 2; do
python bench.py --config C5 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/b5_def_$r.json 2>/dev/null
PINT_LIB=$PWD/paper_2007_13125_b200/libpint_cqf3.so python bench.py --config C5 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/b5_m3_$r.json 2>/dev/null
for v in def m3; do python -c "import json;d=json.load(open('gpurun_out/b5_${v}_$r.json'));print('$v', d['ms_per_step'], d['roofline']['passes']['tpass_ms'])"; done
done
timeout 600 ncu --set full --import-source on -k regex:tpass_cq_fused -c 1 -o gpurun_out/prof_cqf_v5 python bench.py --config C5 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_cqf_v5.log 2>&1
tail -1 gpurun_out/ncu_cqf_v5.log
