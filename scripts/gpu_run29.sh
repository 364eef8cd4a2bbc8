mkdir -p gpurun_out
PINT_LIB=$PWD/paper_2007_13125_b200/libpint_modal2.so timeout 600 python bench.py --modal --no-cpu --no-e2e > gpurun_out/bench29_modal2.json 2> gpurun_out/bench29_modal2.err
