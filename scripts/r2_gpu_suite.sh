# GPU suite (not slow) + bench lines for every config + ncu of the CQ T-pass.  Usage: bash scripts/r2_gpu_suite.sh TAG
T=${1:-v}
python -m pytest tests -x -q -m "gpu and not slow" > gpurun_out/pytest_$T.log 2>&1
tail -3 gpurun_out/pytest_$T.log
for C in C1 C2 C3 C5 C4; do
  timeout 900 python bench.py --config $C --steps 10 --warmup 3 --no-cpu > gpurun_out/b_${T}_$C.json 2> gpurun_out/b_${T}_$C.err
  python -c "import json;d=json.load(open('gpurun_out/b_${T}_$C.json'));print('$C', d['ms_per_step'], d['roofline']['passes'], d.get('materialize'), d['e2e']['value'] if d.get('e2e') else None)"
done
timeout 600 ncu --set full --import-source on -k regex:tpass_cq_fused -c 1 -o gpurun_out/prof_cqf_$T python bench.py --config C5 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_cqf_$T.log 2>&1
tail -1 gpurun_out/ncu_cqf_$T.log
