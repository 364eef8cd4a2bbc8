mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "modal" > gpurun_out/pytest_gpu28a.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu28a.log
timeout 600 python bench.py --modal --no-cpu > gpurun_out/bench28_modal.json 2> gpurun_out/bench28_modal.err
timeout 600 python bench.py --modal --real --no-cpu --no-e2e > gpurun_out/bench28_modal_real.json 2> gpurun_out/bench28_modal_real.err
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:wr_modal_kernel -s 3 -c 1 -o gpurun_out/prof_modal_v1 -f python bench.py --modal --steps 1 --warmup 3 --no-e2e --no-cpu --mx 127 > gpurun_out/ncu_full28.log 2>&1
