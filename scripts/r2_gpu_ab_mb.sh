# S-pass pair kernel occupancy: default (4 CTAs/SM) vs 5 and 6 (ab/libpint_mb5.so, ab/libpint_mb6.so)
for r in 1 2; do
 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/abmb_def_$r.json 2>/dev/null
 for v in mb5 mb6; do PINT_LIB=$PWD/ab/libpint_$v.so python bench.py --config C5 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/abmb_${v}_$r.json 2>/dev/null; done
 for v in def mb5 mb6; do python -c "import json;d=json.load(open('gpurun_out/abmb_${v}_$r.json'));print('C5 $v', d['ms_per_step'], d['roofline']['passes']['spass_ms'])"; done
done
