# fail loudly if the library is stale
python -c "
import os; from paper_2007_13125_b200 import build as b
lib=b.LIB; assert os.path.getmtime(lib) >= b._newest_dep(), 'stale libpint.so'" || exit 3
python -m pytest tests -x -q -s -m "gpu and not slow" -k "modal_window_monitor" 2>&1 | grep -E "modal|passed|failed" > gpurun_out/t7m.log
python -m pytest tests -x -q -m "gpu and not slow" -k "cq or c5 or C5 or full or random_complex or residual or modal or slabs or device_loop or divergence or graph" > gpurun_out/t7.log 2>&1
tail -2 gpurun_out/t7.log
for r in 1 2; do
python bench.py --config C5 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/b7_$r.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/b7_$r.json'));print('C5', d['ms_per_step'], d['roofline']['passes']['tpass_ms'])"
done
python bench.py --config C4 --modal --steps 5 --warmup 3 --no-cpu > gpurun_out/b7_c4modal.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/b7_c4modal.json'));print('C4 modal', d['ms_per_step'], d['e2e']['what'], d['last_update'])"
timeout 600 ncu --set full --import-source on -k regex:tpass_cq_fused -c 1 -o gpurun_out/prof_cqf_v7 python bench.py --config C5 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_cqf_v7.log 2>&1
tail -1 gpurun_out/ncu_cqf_v7.log
