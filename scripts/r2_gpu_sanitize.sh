python -c "
import os; from paper_2007_13125_b200 import build as b
assert os.path.getmtime(b.LIB) >= b._newest_dep(), 'stale libpint.so'" || exit 3
mkdir -p gpurun_out/san
python scripts/sanitize_cases.py > gpurun_out/san/plain.log 2>&1; echo "plain rc=$?"; tail -2 gpurun_out/san/plain.log
for tool in memcheck racecheck synccheck; do
  timeout -s KILL 1500 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 python scripts/sanitize_cases.py > gpurun_out/san/$tool.log 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/san/$tool.log
done
