# the checked build (device-side bounds / protocol assertions; -DPINT_CHECK) on every kernel family
export PINT_LIB=$PWD/ab/libpint_check.so
mkdir -p gpurun_out/chk
timeout -s KILL 900 python scripts/sanitize_cases.py > gpurun_out/chk/cases.log 2>&1; echo "cases rc=$?"; tail -2 gpurun_out/chk/cases.log
timeout -s KILL 1800 python -m pytest tests -q -m "gpu and not slow" -x > gpurun_out/chk/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/chk/pytest.log
