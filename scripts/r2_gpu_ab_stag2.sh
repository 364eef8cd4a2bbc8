# CQ T-pass stagger point: after transform 1 (default), 0, 2, or no stagger
mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m "gpu and not slow" -k "c5 or cq" 2>&1 | tail -1
for r in 1 2; do
 for v in def x0 x2 nost; do
  L=""; [ $v != def ] && L="PINT_LIB=$PWD/ab/libpint_$v.so"
  env $L timeout 300 python bench.py --config C5 --no-cpu --no-e2e > gpurun_out/abst2_${v}_$r.json 2>>gpurun_out/abst2.err
  python -c "import json;a=json.load(open('gpurun_out/abst2_${v}_$r.json'));p=a['roofline']['passes'];print('$v C5', a['ms_per_step'], p['tpass_ms'], p['spass_ms'])"
 done
done
