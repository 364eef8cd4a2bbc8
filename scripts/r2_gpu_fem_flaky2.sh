# zero-filled plan allocations: the dirty-memory regression test (fix and, for contrast, HEAD), then the subset that failed
mkdir -p gpurun_out
timeout 300 python -m pytest tests -q -s -m gpu -k "dirty_memory" 2>&1 | tail -3
PINT_LIB=$PWD/ab/libpint_head.so timeout 300 python -m pytest tests -q -s -m gpu -k "dirty_memory" 2>&1 | tail -3
timeout 900 python -m pytest tests -x -q -s -m "gpu" -k "c1 or c2_sweep or c3 or random_complex or graph or device_loop or unread or pulse or newton or c4_full or c4_window or residual or initial_guess or slabs or dense or real or modal" > gpurun_out/flaky_fix.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/flaky_fix.log; grep -a "solve status" gpurun_out/flaky_fix.log | head -3
