# full GPU suite (incl. slow full-size parity) + measurement set.  Usage: bash scripts/r2_gpu_full.sh TAG
T=${1:-f}
python -c "
import os; from paper_2007_13125_b200 import build as b
assert os.path.getmtime(b.LIB) >= b._newest_dep(), 'stale libpint.so'" || exit 3
mkdir -p gpurun_out/$T
timeout -s KILL 2400 python -m pytest tests -q -m gpu -s > gpurun_out/$T/pytest_gpu_full.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/$T/pytest_gpu_full.log
bash scripts/r2_measure.sh $T
