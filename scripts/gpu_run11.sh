mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench11.json 2> gpurun_out/bench11.err
timeout 600 python bench.py --path stream --no-cpu --no-e2e > gpurun_out/bench11_stream.json 2> gpurun_out/bench11_stream.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches11.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch11.log 2>&1
for c in C1 C2 C3 C5; do timeout 600 python bench.py --config $c --no-cpu > gpurun_out/bench11_$c.json 2> gpurun_out/bench11_$c.err; done
