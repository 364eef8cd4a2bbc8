# A/B timing of two library builds on the same box (box-to-box spread is ~5 %):
#   python -m paper_2007_13125_b200.build -D SOME_MACRO=1 --lib libpint_variant.so --force
#   mkdir -p ab && mv paper_2007_13125_b200/libpint_variant.so ab/
#   gpurun -- bash scripts/gpu_ab.sh ab/libpint_variant.so "--config C4"
mkdir -p gpurun_out
VAR=$1; ARGS=${2:-}
for r in 1 2; do
  timeout 300 python bench.py $ARGS --no-cpu --no-e2e > gpurun_out/ab_cur_$r.json 2>> gpurun_out/ab.err
  PINT_LIB=$VAR timeout 300 python bench.py $ARGS --no-cpu --no-e2e > gpurun_out/ab_var_$r.json 2>> gpurun_out/ab.err
done
