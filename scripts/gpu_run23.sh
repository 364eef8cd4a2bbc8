mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench23.json 2> gpurun_out/bench23.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench23_ref.json 2> gpurun_out/bench23_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches23.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch23.log 2>&1
for c in C1 C2 C3 C5; do timeout 600 python bench.py --config $c --no-cpu > gpurun_out/bench23_$c.json 2> gpurun_out/bench23_$c.err; done
timeout 600 python bench.py --path stream --no-cpu --no-e2e > gpurun_out/bench23_stream.json 2> gpurun_out/bench23_stream.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke23.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke23.log
