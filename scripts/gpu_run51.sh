mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/final51_C4.json 2> gpurun_out/final51.err
for c in C1 C2 C3 C5; do timeout 600 python bench.py --config $c > gpurun_out/final51_$c.json 2>> gpurun_out/final51.err; done
timeout 600 python bench.py --path stream --no-cpu > gpurun_out/final51_stream.json 2>> gpurun_out/final51.err
timeout 600 python bench.py --modal --no-cpu > gpurun_out/final51_modal.json 2>> gpurun_out/final51.err
timeout 600 python bench.py --real --no-cpu > gpurun_out/final51_real.json 2>> gpurun_out/final51.err
timeout 600 python bench.py --modal --real --no-cpu > gpurun_out/final51_modal_real.json 2>> gpurun_out/final51.err
timeout 600 python bench.py --config C5 --modal --no-cpu > gpurun_out/final51_C5_modal.json 2>> gpurun_out/final51.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/final51_ref.json 2>> gpurun_out/final51.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches51.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu51.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke51.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke51.log
