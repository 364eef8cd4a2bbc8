# A/B: zero-carry sweeps start from the first row (no multiply of the zero state) vs ab/libpint_head.so
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m "gpu and not slow" -k "c1 or c2_sweep or c3 or random_complex or graph or device_loop or pulse or c4_window or residual or slabs or fem or modal or real" > gpurun_out/zi_t.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/zi_t.log
for r in 1 2; do
 for v in def head; do
  L=""; [ $v != def ] && L="PINT_LIB=$PWD/ab/libpint_$v.so"
  for C in C4 C3; do
    env $L timeout 300 python bench.py --config $C --no-cpu --no-e2e > gpurun_out/abzi_${v}_${C}_$r.json 2>>gpurun_out/abzi.err
    python -c "import json;a=json.load(open('gpurun_out/abzi_${v}_${C}_$r.json'));print('$v $C', a['ms_per_step'], a['roofline']['frac'])"
  done
 done
done
