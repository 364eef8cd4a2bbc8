python -c "
import os; from paper_2007_13125_b200 import build as b
assert os.path.getmtime(b.LIB) >= b._newest_dep(), 'stale libpint.so'" || exit 3
python -m pytest tests -x -q -m "gpu and not slow" -k "device_loop or divergence or graph or modal or two_processes" > gpurun_out/t11.log 2>&1
tail -2 gpurun_out/t11.log
for C in C1 C2 C3; do python bench.py --config $C --steps 50 --warmup 5 --no-cpu > gpurun_out/b11_$C.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/b11_$C.json'));print('$C', d['ms_per_step'], d['e2e']['value'], d['e2e']['what'][:60])"; done
