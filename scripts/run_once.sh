set -u
export PYTHONUNBUFFERED=1
T=${TAG:-x}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 600 python bench.py --config c1 --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/${T}_bench_c1.log 2>&1
