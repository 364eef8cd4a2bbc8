# solve tail rework (scan-level skip, store-in-sweep fast tail): parity subset, A/B vs ab/libpint_old.so
mkdir -p gpurun_out
python -c "
import os; from paper_2007_13125_b200 import build as b
assert os.path.getmtime(b.LIB) >= b._newest_dep(), 'stale libpint.so'" || exit 3
timeout 900 python -m pytest tests -x -q -m "gpu" -k "c1 or c2_sweep or c3 or random_complex or graph or device_loop or unread or pulse or newton or c4_full or c4_window or residual or initial_guess or slabs or dense" > gpurun_out/solve_t.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/solve_t.log
for r in 1 2; do
 for v in def old teams; do
  L=""; [ $v != def ] && L="PINT_LIB=$PWD/ab/libpint_$v.so"
  for C in C4 C3; do
    env $L timeout 300 python bench.py --config $C --no-cpu --no-e2e > gpurun_out/abs_${v}_${C}_$r.json 2>>gpurun_out/abs.err
    python -c "import json;a=json.load(open('gpurun_out/abs_${v}_${C}_$r.json'));print('$v $C', a['ms_per_step'], a['roofline']['frac'])"
  done
 done
done
PINT_LIB=$PWD/ab/libpint_sprof2.so timeout 300 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu --no-e2e 2>&1 | grep "pint prof" | head -3
