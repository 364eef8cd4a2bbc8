python -c "
import os; from paper_2007_13125_b200 import build as b
assert os.path.getmtime(b.LIB) >= b._newest_dep(), 'stale libpint.so'" || exit 3
python -m pytest tests -x -q -s -m "gpu and not slow" -k "fem2d" 2>&1 | grep -E "fem2d|example3|heat_k4|cq_k1|passed|failed|Error|error" > gpurun_out/t10f.log
python -m pytest tests -x -q -m "gpu and not slow" > gpurun_out/t10.log 2>&1
tail -3 gpurun_out/t10.log
