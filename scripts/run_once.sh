# scratch driver for one gpurun call (edited per experiment): A/B of build/libsb_head.so vs the tree
set -u
export PYTHONUNBUFFERED=1
T=${TAG:-x}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 900 python -m pytest tests -m "gpu and not slow" -q -x 2>&1 | tail -30 > gpurun_out/${T}_tests.log
for c in c2 c3 c1 c4; do
  for r in 1 2; do
  SB_LIB_PATH=$PWD/build/libsb_head.so timeout 600 python bench.py --config $c --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/${T}_A${r}_$c.log 2>&1
  timeout 600 python bench.py --config $c --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/${T}_B${r}_$c.log 2>&1
  done
done
