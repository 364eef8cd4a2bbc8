# Round-2 measurement set on one B200 (gpurun -- bash scripts/r2_measure.sh TAG): bench lines for every
# config/variant, the reference arm, the ncu launch lists of the C4 and C5 benches, modal traffic, smoke.
T=${1:-m}
python -c "
import os; from paper_2007_13125_b200 import build as b
assert os.path.getmtime(b.LIB) >= b._newest_dep(), 'stale libpint.so'" || exit 3
o=gpurun_out/$T; mkdir -p $o
timeout 900 python bench.py > $o/C4.json 2> $o/err.log
for c in C1 C2 C3 C5; do timeout 600 python bench.py --config $c > $o/$c.json 2>> $o/err.log; done
timeout 600 python bench.py --config C3 --e2e-full --no-cpu > $o/C3_e2efull.json 2>> $o/err.log
timeout 600 python bench.py --config C5 --e2e-full --no-cpu > $o/C5_e2efull.json 2>> $o/err.log
timeout 600 python bench.py --path stream --no-cpu > $o/C4_stream.json 2>> $o/err.log
timeout 600 python bench.py --modal --no-cpu > $o/C4_modal.json 2>> $o/err.log
timeout 600 python bench.py --real --no-cpu > $o/C4_real.json 2>> $o/err.log
timeout 600 python bench.py --modal --real --no-cpu > $o/C4_modal_real.json 2>> $o/err.log
timeout 600 python bench.py --config C5 --modal --no-cpu > $o/C5_modal.json 2>> $o/err.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $o/ref.json 2>> $o/err.log
timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu > $o/C4_gpus2.json 2> $o/gpus2.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/launches_C4.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $o/ncu_launch_C4.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/launches_C5.csv python bench.py --config C5 --steps 2 --warmup 3 --no-e2e --no-cpu > $o/ncu_launch_C5.log 2>&1
timeout 900 ncu --set full --import-source on -k regex:wr_modal_kernel -c 1 -o $o/prof_modal python bench.py --modal --mx 127 --steps 1 --warmup 3 --no-e2e --no-cpu > $o/ncu_modal.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; echo "smoke rc=$?" >> $o/smoke.log
for f in $o/*.json; do python -c "
import json,sys; d=json.load(open('$f')); r=d.get('roofline') or {}; e=d.get('e2e') or {}
print('$f'.split('/')[-1], d.get('ms_per_step'), '%.3e'%d['value'], r.get('bound'), r.get('frac'), '%.3e'%(e.get('value') or 0), e.get('converged'))" 2>/dev/null; done
