python -c "
import os; from paper_2007_13125_b200 import build as b
assert os.path.getmtime(b.LIB) >= b._newest_dep(), 'stale libpint.so'" || exit 3
python -m pytest tests -x -q -m "gpu and not slow" -k "cq or c5 or C5 or full or random_complex or residual or modal or slabs or u0_zero or fem or dense or two_processes" > gpurun_out/t21.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/t21.log
python bench.py --config C5 --steps 10 --warmup 3 --no-cpu > gpurun_out/b21_C5.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/b21_C5.json'));print('C5', d['ms_per_step'], d['e2e'])"
