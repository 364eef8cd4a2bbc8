python -c "
import os; from paper_2007_13125_b200 import build as b
assert os.path.getmtime(b.LIB) >= b._newest_dep(), 'stale libpint.so'" || exit 3
timeout -s KILL 300 python -m pytest tests -x -q -m "gpu and not slow" -k "device_loop or divergence or graph_replay or wr_run or c1 or c2_sweep" > gpurun_out/t14.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/t14.log
for C in C1 C2; do timeout -s KILL 120 python bench.py --config $C --steps 50 --warmup 5 --no-cpu > gpurun_out/b14_$C.json 2>gpurun_out/b14_$C.err; python -c "import json;d=json.load(open('gpurun_out/b14_$C.json'));print('$C', d['ms_per_step'], d['e2e']['value'], d['gpu_launches'])"; done
