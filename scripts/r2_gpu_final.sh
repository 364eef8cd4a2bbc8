# session-2 measurement set: full GPU suite, bench set (r2_measure.sh), full-size ncu capture of the C4 fused kernel
T=${1:-f3}
bash scripts/r2_gpu_full.sh $T
timeout 900 ncu --set full --import-source on --clock-control none -k regex:wr_fused_kernel -s 1 -c 1 -o gpurun_out/$T/prof_fused_c4full -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/$T/ncu_fused_c4full.log 2>&1
ls -la gpurun_out/$T/*.ncu-rep
