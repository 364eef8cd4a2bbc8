# final-code profiles (session 3): ncu --set full of the C5 S-pass pair kernel; launch lists of the C4 / C5 bench commands
python -c "
import os; from paper_2007_13125_b200 import build as b
assert os.path.getmtime(b.LIB) >= b._newest_dep(), 'stale libpint.so'" || exit 3
o=gpurun_out/p6; mkdir -p $o
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spass_pair_kernel -s 2 -c 1 -o $o/prof_spass_f6 -f python bench.py --config C5 --steps 1 --warmup 3 --no-cpu --no-e2e > $o/ncu_spass.log 2>&1
echo "ncu spass rc=$?"; tail -2 $o/ncu_spass.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/launches_C4.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $o/ncu_launch_C4.log 2>&1
echo "ncu C4 launches rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/launches_C5.csv python bench.py --config C5 --steps 2 --warmup 3 --no-e2e --no-cpu > $o/ncu_launch_C5.log 2>&1
echo "ncu C5 launches rc=$?"
