set -u
export PYTHONUNBUFFERED=1
T=${TAG:-x}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
for v in 0 1 2 3; do
  SB_ROWS_VARIANT=$v timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "small_parity" > gpurun_out/${T}_v${v}_tests.log 2>&1
  for c in c2 c1 c4; do SB_ROWS_VARIANT=$v timeout 600 python bench.py --config $c --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/${T}_v${v}_$c.log 2>&1; done
done
