python -c "
import os; from paper_2007_13125_b200 import build as b
assert os.path.getmtime(b.LIB) >= b._newest_dep(), 'stale libpint.so'" || exit 3
for C in C1 C2; do
timeout 600 ncu --set full --import-source on -k wr_loop_kernel -c 1 -o gpurun_out/prof_loop_$C python bench.py --config $C --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_loop_$C.log 2>&1
done
tail -2 gpurun_out/ncu_loop_C2.log
