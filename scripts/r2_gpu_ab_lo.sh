# A/B: solve load order and dft8 zero-input pruning (default both on) vs variants in ab/
mkdir -p gpurun_out
for r in 1 2; do
 for v in def nolo nodz nolodz; do
  L=""; [ $v != def ] && L="PINT_LIB=$PWD/ab/libpint_$v.so"
  for C in C4 C3; do
    env $L timeout 300 python bench.py --config $C --no-cpu --no-e2e > gpurun_out/ablo_${v}_${C}_$r.json 2>>gpurun_out/ablo.err
    python -c "import json;a=json.load(open('gpurun_out/ablo_${v}_${C}_$r.json'));print('$v $C', a['ms_per_step'], a['roofline']['frac'])"
  done
 done
done
