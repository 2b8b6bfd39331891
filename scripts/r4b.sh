set -u
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r4b_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "sv or deterministic or shards or workspace_reuse or identical" > gpurun_out/r4b_tests.log 2>&1
tail -5 gpurun_out/r4b_tests.log
for c in c2 c1; do timeout 300 python bench.py --config $c --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/r4b_bench_$c.log 2>&1; done
