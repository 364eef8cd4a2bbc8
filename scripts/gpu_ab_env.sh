# A/B of an environment switch on the same box: gpurun -- bash scripts/gpu_ab_env.sh PINT_CQ_MONO=1 "--config C5"
mkdir -p gpurun_out
ENVV=$1; ARGS=${2:-}
for r in 1 2; do
  timeout 300 python bench.py $ARGS --no-cpu --no-e2e > gpurun_out/abe_cur_$r.json 2>> gpurun_out/abe.err
  env $ENVV timeout 300 python bench.py $ARGS --no-cpu --no-e2e > gpurun_out/abe_var_$r.json 2>> gpurun_out/abe.err
done
