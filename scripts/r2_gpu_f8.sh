# verification on the restored container (session 4): full GPU suite, C4 / C5 / C3 bench lines, smoke
T=f8
python -c "
import os; from paper_2007_13125_b200 import build as b
assert os.path.getmtime(b.LIB) >= b._newest_dep(), 'stale libpint.so'" || exit 3
o=gpurun_out/$T; mkdir -p $o
timeout -s KILL 2400 python -m pytest tests -q -m gpu -s > $o/pytest_gpu_full.log 2>&1
echo "pytest rc=$?"; tail -2 $o/pytest_gpu_full.log
timeout 900 python bench.py > $o/C4.json 2> $o/err.log
timeout 600 python bench.py --config C5 > $o/C5.json 2>> $o/err.log
timeout 600 python bench.py --config C3 > $o/C3.json 2>> $o/err.log
python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; echo "smoke rc=$?" >> $o/smoke.log
for f in $o/*.json; do python -c "
import json,sys; d=json.load(open('$f')); r=d.get('roofline') or {}; e=d.get('e2e') or {}
print('$f'.split('/')[-1], d.get('ms_per_step'), '%.3e'%d['value'], r.get('bound'), r.get('frac'), '%.3e'%(e.get('value') or 0), e.get('converged'))" 2>/dev/null; done
# launch list of the default bench command (run above without ncu, exit 0)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/launches_C4.csv python bench.py --steps 3 --warmup 3 > $o/ncu_C4.log 2>&1; echo "ncu rc=$?"
