# CQ T-pass: the two tile groups staggered by half a tile (ab/libpint_stag.so) vs default; parity on the variant
mkdir -p gpurun_out
PINT_LIB=$PWD/ab/libpint_stag.so timeout 600 python -m pytest tests -x -q -m "gpu and not slow" -k "c5 or cq" 2>&1 | tail -1
for r in 1 2; do
 for v in def stag; do
  L=""; [ $v != def ] && L="PINT_LIB=$PWD/ab/libpint_$v.so"
  env $L timeout 300 python bench.py --config C5 --no-cpu --no-e2e > gpurun_out/abst_${v}_$r.json 2>>gpurun_out/abst.err
  python -c "import json;a=json.load(open('gpurun_out/abst_${v}_$r.json'));p=a['roofline']['passes'];print('$v C5', a['ms_per_step'], p['tpass_ms'], p['spass_ms'])"
 done
done
