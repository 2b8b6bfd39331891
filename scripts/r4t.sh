set -u
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r4t_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_confidence.py -m "gpu and not slow" -x -q -p no:cacheprovider > gpurun_out/r4t_tests.log 2>&1
tail -2 gpurun_out/r4t_tests.log
for r in 1 2 3; do timeout 300 python bench.py --config c2 --steps 30 --no-e2e --no-cpu-baseline 2>/dev/null | grep "^{" | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('c2', j['ms_per_step'], j['value'])"; done
SB_ASTEP=1 timeout 300 python scripts/astep_fixed.py 64 2>&1 | tail -1
export SB_LIB_PATH=$PWD/build/lib_trace.so
timeout 300 python scripts/astep_trace.py c2 > gpurun_out/r4t_astep_c2.txt 2>&1
