set -u
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2h_build.log 2>&1
for c in c2 c1one c3; do SB_LIB_PATH=$PWD/build/lib_trace.so timeout 300 python scripts/step_trace.py $c > gpurun_out/r2h_trace_$c.log 2>&1; done
timeout 900 python -m pytest tests -m "gpu and not slow" -q -p no:cacheprovider 2>&1 | tail -4 > gpurun_out/r2h_tests.log
