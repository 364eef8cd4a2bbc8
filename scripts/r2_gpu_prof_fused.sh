# ncu --set full of the C4 fused kernel at FULL size (the bench configuration: traffic per launch)
python -c "
import os; from paper_2007_13125_b200 import build as b
assert os.path.getmtime(b.LIB) >= b._newest_dep(), 'stale libpint.so'" || exit 3
timeout 900 ncu --set full --import-source on -k wr_fused_kernel -c 1 -o gpurun_out/prof_fused_c4full python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_fused_c4full.log 2>&1
tail -2 gpurun_out/ncu_fused_c4full.log
