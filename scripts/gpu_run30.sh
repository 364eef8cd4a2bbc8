mkdir -p gpurun_out
PINT_LIB=$PWD/paper_2007_13125_b200/libpint_modal3.so timeout 600 python bench.py --modal --no-cpu --no-e2e > gpurun_out/bench30_modal3.json 2> gpurun_out/bench30_modal3.err
timeout 600 python -m pytest tests -m gpu -q -x -k "modal" > gpurun_out/pytest_gpu30.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu30.log
timeout 600 python bench.py --modal --no-cpu > gpurun_out/bench30_modal.json 2> gpurun_out/bench30_modal.err
timeout 600 python bench.py --modal --real --no-cpu --no-e2e > gpurun_out/bench30_modal_real.json 2> gpurun_out/bench30_modal_real.err
