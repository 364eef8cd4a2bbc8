# CQ T-pass: DFT32 radix-2 stage as FMA butterflies (PINT_CQ_FMABF); parity subset on the variant, A/B on C5
mkdir -p gpurun_out/fb
V=PINT_LIB=$PWD/paper_2007_13125_b200/libpint_fmabf.so
env $V timeout 900 python -m pytest tests -x -q -m "gpu and not slow" -k "cq or c5 or C5 or full or random_complex or residual" > gpurun_out/fb/t.log 2>&1
echo "pytest(fmabf) rc=$?"; tail -2 gpurun_out/fb/t.log
for r in 1 2 3; do
 for v in def fmabf; do
  L=""; [ $v != def ] && L=$V
  env $L timeout 300 python bench.py --config C5 --no-cpu --no-e2e > gpurun_out/fb/${v}_C5_$r.json 2>>gpurun_out/fb/err.log
  python -c "
import json
a=json.load(open('gpurun_out/fb/${v}_C5_$r.json')); p=a['roofline'].get('passes'); print('$v', round(a['ms_per_step'],4), round(p['tpass_ms'],4), round(p['spass_ms'],4))"
 done
done
