# S-pass pair solve: value-form (AF, default) vs u-form only (ab/libpint_noaf.so)
for r in 1 2; do
 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/abaf_def_$r.json 2>/dev/null
 PINT_LIB=$PWD/ab/libpint_noaf.so python bench.py --config C5 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/abaf_noaf_$r.json 2>/dev/null
 for v in def noaf; do python -c "import json;d=json.load(open('gpurun_out/abaf_${v}_$r.json'));print('C5 $v', d['ms_per_step'], d['roofline']['passes']['spass_ms'])"; done
 python bench.py --path stream --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/abafs_def_$r.json 2>/dev/null
 PINT_LIB=$PWD/ab/libpint_noaf.so python bench.py --path stream --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/abafs_noaf_$r.json 2>/dev/null
 for v in def noaf; do python -c "import json;d=json.load(open('gpurun_out/abafs_${v}_$r.json'));print('C4s $v', d['ms_per_step'], d['roofline']['passes']['spass_ms'])"; done
done
python -m pytest tests/test_gpu_parity.py -x -q -k "c2 or cq or stream or random_complex or spass" 2>&1 | tail -3
