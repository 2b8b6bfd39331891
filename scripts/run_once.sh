set -u
export PYTHONUNBUFFERED=1
T=${TAG:-x}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
for c in c3 c2; do timeout 600 python bench.py --config $c --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/${T}_$c.log 2>&1; done
