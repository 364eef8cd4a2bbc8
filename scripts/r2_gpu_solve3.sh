# solve loads in consumption order; A/B g-form (default) vs ab/libpint_nog.so vs ab/libpint_old.so (round-2 HEAD)
mkdir -p gpurun_out
python -c "
import os; from paper_2007_13125_b200 import build as b
assert os.path.getmtime(b.LIB) >= b._newest_dep(), 'stale libpint.so'" || exit 3
timeout 900 python -m pytest tests -q -m "gpu and not slow" > gpurun_out/solve3_t.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/solve3_t.log; grep FAILED gpurun_out/solve3_t.log | head
for r in 1 2; do
 for v in def nog old; do
  L=""; [ $v != def ] && L="PINT_LIB=$PWD/ab/libpint_$v.so"
  for C in C4 C3; do
    env $L timeout 300 python bench.py --config $C --no-cpu --no-e2e > gpurun_out/abs3_${v}_${C}_$r.json 2>>gpurun_out/abs3.err
    python -c "import json;a=json.load(open('gpurun_out/abs3_${v}_${C}_$r.json'));print('$v $C', a['ms_per_step'], a['roofline']['frac'])"
  done
 done
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:wr_fused -s 1 -c 1 -o gpurun_out/prof_s3 -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --mx 127 > gpurun_out/ncu_s3.log 2>&1
ls -la gpurun_out/prof_s3.ncu-rep
