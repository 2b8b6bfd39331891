set -u
export PYTHONUNBUFFERED=1
T=${TAG:-x}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_next.py -q -x 2>&1 | tail -3 > gpurun_out/${T}_tests.log
for c in kv tree; do timeout 600 python bench.py --config $c --steps 20 > gpurun_out/${T}_bench_$c.log 2>&1; done
