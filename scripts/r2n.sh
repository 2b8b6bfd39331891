set -u
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2n_build.log 2>&1
timeout 900 python -m pytest tests -m "gpu and not slow" -q -p no:cacheprovider 2>&1 | tail -4 > gpurun_out/r2n_tests.log
for c in c4 c2 c3 c1; do timeout 600 python bench.py --config $c --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/r2n_bench_$c.log 2>&1; done
timeout 1500 python -m pytest tests -m "gpu and slow" -q -s -p no:cacheprovider 2>&1 | grep -v "^\s*$" | tail -12 > gpurun_out/r2n_slow.log
