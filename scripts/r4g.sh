set -u
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r4g_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_confidence.py -m gpu -x -q -p no:cacheprovider -k "sv or astep or adaptive or deterministic or shards or workspace_reuse" > gpurun_out/r4g_tests.log 2>&1
tail -3 gpurun_out/r4g_tests.log
for r in 1 2; do timeout 300 python bench.py --config c2 --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/r4g_bench_c2_$r.log 2>&1; done
export SB_LIB_PATH=$PWD/build/lib_trace.so
timeout 300 python scripts/astep_trace.py c2 > gpurun_out/r4g_astep_c2.txt 2>&1
