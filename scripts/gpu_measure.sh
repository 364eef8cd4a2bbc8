# Round-1 measurement set on one B200 (run from the repo root: gpurun -- bash scripts/gpu_measure.sh):
# bench lines for every config/variant, the reference arm, the ncu launch list of the C4 bench, smoke.
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/final_C4.json 2> gpurun_out/final.err
for c in C1 C2 C3 C5; do timeout 600 python bench.py --config $c > gpurun_out/final_$c.json 2>> gpurun_out/final.err; done
timeout 600 python bench.py --path stream --no-cpu > gpurun_out/final_stream.json 2>> gpurun_out/final.err
timeout 600 python bench.py --modal --no-cpu > gpurun_out/final_modal.json 2>> gpurun_out/final.err
timeout 600 python bench.py --real --no-cpu > gpurun_out/final_real.json 2>> gpurun_out/final.err
timeout 600 python bench.py --modal --real --no-cpu > gpurun_out/final_modal_real.json 2>> gpurun_out/final.err
timeout 600 python bench.py --config C5 --modal --no-cpu > gpurun_out/final_C5_modal.json 2>> gpurun_out/final.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/final_ref.json 2>> gpurun_out/final.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke51.log
