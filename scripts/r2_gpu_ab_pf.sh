# S-pass pair kernel: L2 prefetch of the rows one resident wave ahead (PINT_PAIR_PF CTAs); A/B on C5 and C4 streaming
mkdir -p gpurun_out/pf
for r in 1 2; do
 for v in def pf600 pf1200; do
  L=""; [ $v != def ] && L="PINT_LIB=$PWD/paper_2007_13125_b200/libpint_$v.so"
  env $L timeout 300 python bench.py --config C5 --no-cpu --no-e2e > gpurun_out/pf/${v}_C5_$r.json 2>>gpurun_out/pf/err.log
  env $L timeout 300 python bench.py --config C4 --path stream --no-cpu --no-e2e > gpurun_out/pf/${v}_C4s_$r.json 2>>gpurun_out/pf/err.log
  python -c "
import json
for c in ['C5','C4s']:
  a=json.load(open('gpurun_out/pf/${v}_'+c+'_$r.json')); print('$v', c, round(a['ms_per_step'],4), a['roofline'].get('passes'))"
 done
done
