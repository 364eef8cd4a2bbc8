for c in C2 C1; do PINT_LIB=$PWD/ab/libpint_prof.so python bench.py --config $c --steps 20 --warmup 3 --no-cpu --no-e2e 2>&1 | grep -E "pint prof\] loop"; done
for c in C1 C2; do python bench.py --config $c --steps 200 --warmup 5 --no-cpu 2>/dev/null > gpurun_out/fin_$c.json; python -c "import json;d=json.load(open('gpurun_out/fin_$c.json'));print('$c', d['ms_per_step']*1000, 'us', d['e2e']['value'])"; done
python -m pytest tests/test_gpu_parity.py -x -q -k "c1 or c2 or loop or run or diverg or solve" 2>&1 | tail -2
