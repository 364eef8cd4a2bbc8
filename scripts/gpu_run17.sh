mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu17.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu17.log
timeout 300 python bench.py --no-cpu --no-e2e --steps 10 > gpurun_out/bench17_xs.json 2> gpurun_out/bench17_xs.err
PINT_FUSED_NO_XS=1 timeout 300 python bench.py --no-cpu --no-e2e --steps 10 > gpurun_out/bench17_noxs.json 2> gpurun_out/bench17_noxs.err
PINT_LIB=$PWD/paper_2007_13125_b200/libpint_prof.so timeout 300 python bench.py --no-cpu --no-e2e --steps 3 --warmup 1 > gpurun_out/bench17_prof.json 2> gpurun_out/bench17_prof.err
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:wr_fused_kernel -s 3 -c 1 -o gpurun_out/prof_fused_v7 -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --mx 127 > gpurun_out/ncu_full17.log 2>&1
