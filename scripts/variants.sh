#!/bin/bash
# Benchmark k_rows_tma geometry variants (SB_ROWS_VARIANT) on C4 / C1 / C2 and check parity.
TAG=$1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in ${VARIANTS:-0 1 2 3 4}; do
  SB_ROWS_VARIANT=$v timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "small_parity and (V32000 or ragged or K8)" > gpurun_out/${TAG}_v${v}_tests.log 2>&1
  for c in ${CONFIGS:-c4 c1 c2}; do
    SB_ROWS_VARIANT=$v timeout 300 python bench.py --config $c --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_v${v}_$c.log 2>&1
  done
done
