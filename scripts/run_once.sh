set -u
export PYTHONUNBUFFERED=1
T=${TAG:-x}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_next.py -q -x -k spawn 2>&1 | tail -2 > gpurun_out/${T}_tests.log
for r in 1 2; do timeout 600 python bench.py --config spawn --steps 20 > gpurun_out/${T}_bench_spawn_$r.log 2>&1; done
