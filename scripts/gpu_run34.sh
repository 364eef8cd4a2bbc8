mkdir -p gpurun_out
for i in 1 2; do
PINT_LIB=$PWD/paper_2007_13125_b200/libpint_pre.so timeout 300 python bench.py --no-cpu --no-e2e --steps 20 > gpurun_out/bench34_pre_$i.json 2> gpurun_out/bench34_pre_$i.err
timeout 300 python bench.py --no-cpu --no-e2e --steps 20 > gpurun_out/bench34_cur_$i.json 2> gpurun_out/bench34_cur_$i.err
done
timeout 300 python bench.py --real --no-cpu --no-e2e --steps 20 > gpurun_out/bench34_real.json 2> gpurun_out/bench34_real.err
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu34.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu34.log
