# fused heat kernel sub-chains per lane chunk: default NS = 4 vs ab/libpint_ns2.so, ab/libpint_ns8.so (C4, C3)
for r in 1 2; do
 for v in def ns2 ns8; do
  L=""; [ $v != def ] && L="PINT_LIB=$PWD/ab/libpint_$v.so"
  env $L python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/abns_${v}_$r.json 2>/dev/null
  env $L python bench.py --config C3 --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/abns3_${v}_$r.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/abns_${v}_$r.json'));e=json.load(open('gpurun_out/abns3_${v}_$r.json'));print('$v C4', d['ms_per_step'], 'C3', e['ms_per_step'])"
 done
done
python -m pytest tests/test_gpu_parity.py -x -q -k "random_complex" 2>&1 | tail -2
