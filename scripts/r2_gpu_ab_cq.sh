# C5 one-kernel CQ T-pass: working tree (default lib) vs ab/libpint_old.so
for r in 1 2; do
 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/abcq_new_$r.json 2>/dev/null
 PINT_LIB=$PWD/ab/libpint_old.so python bench.py --config C5 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/abcq_old_$r.json 2>/dev/null
 for v in new old; do python -c "import json;d=json.load(open('gpurun_out/abcq_${v}_$r.json'));print('C5 $v', d['ms_per_step'], d['roofline']['passes'])"; done
done
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "cq or c5 or full_update or random_complex" 2>&1 | tail -3
if [ -n "$NCU" ]; then
ncu --set full --clock-control none --import-source on -k tpass_cq_fused_kernel -s 2 -c 1 -o gpurun_out/prof_cqf_$NCU -f python bench.py --config C5 --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_cq.log 2>&1
fi
