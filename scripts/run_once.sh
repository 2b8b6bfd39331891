set -u
export PYTHONUNBUFFERED=1
T=${TAG:-x}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
for r in 1 2 3; do for v in 0 2 1; do
  SB_ROWS_VARIANT=$v timeout 600 python bench.py --config c4 --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/${T}_r${r}_v${v}_c4.log 2>&1
done; done
for v in 0 2; do for c in c1 c2 c3; do SB_ROWS_VARIANT=$v timeout 600 python bench.py --config $c --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/${T}_v${v}_$c.log 2>&1; done; done
