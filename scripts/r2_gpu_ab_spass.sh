for r in 1 2; do
 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab22_def_$r.json 2>/dev/null
 for v in lpc4 lpc8; do PINT_LIB=$PWD/ab/libpint_$v.so python bench.py --config C5 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab22_${v}_$r.json 2>/dev/null; done
 for v in def lpc4 lpc8; do python -c "import json;d=json.load(open('gpurun_out/ab22_${v}_$r.json'));print('$v', d['ms_per_step'], d['roofline']['passes']['spass_ms'])"; done
 python bench.py --path stream --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab22s_def_$r.json 2>/dev/null
 PINT_LIB=$PWD/ab/libpint_lpc4.so python bench.py --path stream --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab22s_lpc4_$r.json 2>/dev/null
 for v in def lpc4; do python -c "import json;d=json.load(open('gpurun_out/ab22s_${v}_$r.json'));print('C4s $v', d['ms_per_step'], d['roofline']['passes']['spass_ms'])"; done
done
