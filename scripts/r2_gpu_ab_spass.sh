# S-pass: in-warp scan levels with |a^{C 2^i}| < 2^-64 skipped; A/B vs ab/libpint_head.so on C5 (and C4 stream)
mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m "gpu and not slow" -k "c5 or cq or stream or random_complex" > gpurun_out/sp_t.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/sp_t.log
for r in 1 2; do
 for v in def head; do
  L=""; [ $v != def ] && L="PINT_LIB=$PWD/ab/libpint_$v.so"
  env $L timeout 300 python bench.py --config C5 --no-cpu --no-e2e > gpurun_out/absp_${v}_C5_$r.json 2>>gpurun_out/absp.err
  env $L timeout 300 python bench.py --config C4 --path stream --no-cpu --no-e2e > gpurun_out/absp_${v}_C4s_$r.json 2>>gpurun_out/absp.err
  python -c "
import json
for c in ['C5','C4s']:
  a=json.load(open('gpurun_out/absp_${v}_'+c+'_$r.json')); print('$v', c, a['ms_per_step'], a['roofline'].get('passes'))"
 done
done
