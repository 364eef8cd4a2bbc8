for r in 1 2; do for C in C1 C2; do
 python bench.py --config $C --steps 50 --warmup 5 --no-cpu --no-e2e > gpurun_out/ab23_def_${C}_$r.json 2>/dev/null
 PINT_LIB=$PWD/ab/libpint_spin.so python bench.py --config $C --steps 50 --warmup 5 --no-cpu --no-e2e > gpurun_out/ab23_spin_${C}_$r.json 2>/dev/null
 python -c "import json;a=json.load(open('gpurun_out/ab23_def_${C}_$r.json'));b=json.load(open('gpurun_out/ab23_spin_${C}_$r.json'));print('$C sleep40', a['ms_per_step'], 'spin', b['ms_per_step'])"
done; done
