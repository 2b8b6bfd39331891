set -u
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r4j_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_confidence.py tests/test_gpu_laws.py -m "gpu and not slow" -x -q -p no:cacheprovider > gpurun_out/r4j_tests.log 2>&1
tail -3 gpurun_out/r4j_tests.log
for n in 4 1 2 4 1; do SB_ASTEP_PARTS=$n timeout 300 python bench.py --config c2 --steps 30 --no-e2e --no-cpu-baseline | grep "^{" | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(\"parts $n\", j[\"ms_per_step\"], j[\"value\"])"; done
export SB_LIB_PATH=$PWD/build/lib_trace.so
timeout 300 python scripts/astep_trace.py c2 > gpurun_out/r4j_astep_c2.txt 2>&1
