python -c "
import os; from paper_2007_13125_b200 import build as b
assert os.path.getmtime(b.LIB) >= b._newest_dep(), 'stale libpint.so'" || exit 3
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launch13_modal.csv python bench.py --modal --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
for C in C1 C2; do python bench.py --config $C --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/b13_$C.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/b13_$C.json'));print('$C', d['ms_per_step'])"; done
python bench.py --config C5 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/b13_C5.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/b13_C5.json'));print('C5', d['ms_per_step'], d['roofline'])"
