# ncu capture of the C5 S-pass pair kernel (tag $1)
ncu --set full --clock-control none --import-source on -k regex:spass_pair_kernel -s 2 -c 1 -o gpurun_out/prof_spass_$1 -f python bench.py --config C5 --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_spass.log 2>&1
tail -3 gpurun_out/ncu_spass.log
