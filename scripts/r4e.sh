set -u
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r4e_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_confidence.py -m gpu -x -q -p no:cacheprovider -k "sv or deterministic or shards or workspace_reuse or identical or adaptive" > gpurun_out/r4e_tests.log 2>&1
tail -5 gpurun_out/r4e_tests.log
for c in c2 c1; do timeout 300 python bench.py --config $c --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/r4e_bench_$c.log 2>&1; done
export SB_LIB_PATH=$PWD/build/lib_trace.so
timeout 300 python scripts/sv_trace.py c2 > gpurun_out/r4e_sv_c2.txt 2>&1
timeout 300 python scripts/sv_trace.py c1one > gpurun_out/r4e_sv_c1.txt 2>&1
