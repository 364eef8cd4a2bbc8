python -c "
import os; from paper_2007_13125_b200 import build as b
assert os.path.getmtime(b.LIB) >= b._newest_dep(), 'stale libpint.so'" || exit 3
python -m pytest tests -x -q -m "gpu" -k "c1 or c2_sweep or c3 or random_complex or graph or device_loop or unread or pulse or real_data or newton or c4_full or c4_window or residual or initial_guess or slabs or two_processes" > gpurun_out/t19.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/t19.log
for r in 1 2; do
 for C in C4 C3; do
  timeout 300 python bench.py --config $C --no-cpu --no-e2e > gpurun_out/ab19_new_${C}_$r.json 2>/dev/null
  PINT_LIB=$PWD/ab/libpint_head.so timeout 300 python bench.py --config $C --no-cpu --no-e2e > gpurun_out/ab19_old_${C}_$r.json 2>/dev/null
  python -c "import json;a=json.load(open('gpurun_out/ab19_new_${C}_$r.json'));b=json.load(open('gpurun_out/ab19_old_${C}_$r.json'));print('$C new', a['ms_per_step'], 'old', b['ms_per_step'])"
 done
done
