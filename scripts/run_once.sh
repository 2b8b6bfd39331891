set -u
export PYTHONUNBUFFERED=1
T=${TAG:-x}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 900 python -m pytest tests -m "gpu and not slow" -q -x 2>&1 | tail -3 > gpurun_out/${T}_tests.log
timeout 300 python bench.py --config hrad --steps 30 --no-cpu-baseline > gpurun_out/${T}_hrad.log 2>&1
