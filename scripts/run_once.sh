set -u
export PYTHONUNBUFFERED=1
T=${TAG:-x}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 900 python -m pytest tests -m "gpu" -q -x 2>&1 | tail -30 > gpurun_out/${T}_tests.log
for c in c2 c1 c3 c4 c5; do timeout 600 python bench.py --config $c --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/${T}_bench_$c.log 2>&1; done
