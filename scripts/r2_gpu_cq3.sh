# CQ T-pass: parity subset, C5 bench x2, ncu; modal monitor tests
python -m pytest tests -x -q -m "gpu and not slow" -k "cq or c5 or C5 or full or random_complex or residual or modal or slabs or device_loop or divergence" > gpurun_out/t6.log 2>&1
tail -2 gpurun_out/t6.log
for r in 1 2; do
python bench.py --config C5 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/b6_$r.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/b6_$r.json'));print('C5', d['ms_per_step'], d['roofline']['passes']['tpass_ms'])"
done
for C in C1 C2; do python bench.py --config $C --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/b6_$C.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/b6_$C.json'));print('$C', d['ms_per_step'])"; done
timeout 600 ncu --set full --import-source on -k regex:tpass_cq_fused -c 1 -o gpurun_out/prof_cqf_v6 python bench.py --config C5 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_cqf_v6.log 2>&1
tail -1 gpurun_out/ncu_cqf_v6.log
