# reproduce the once-seen test_fem_and_modal_1d[fem_63_bdf2] non-convergence: the subset of that run, twice
mkdir -p gpurun_out
for r in 1 2; do
timeout 900 python -m pytest tests -x -q -s -m "gpu" -k "c1 or c2_sweep or c3 or random_complex or graph or device_loop or unread or pulse or newton or c4_full or c4_window or residual or initial_guess or slabs or dense or real or modal" > gpurun_out/flaky_$r.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/flaky_$r.log; grep -a "fem_63\|solve status" gpurun_out/flaky_$r.log | head -5
done
