#!/bin/bash
# Round-2 GPU session: build, fast GPU tests, a set of bench lines.
# usage: scripts/r2_bench.sh TAG "c4 c2 c1" [tests] [slow]
set -u
TAG=$1; CFGS=${2:-"c4 c2"}; shift 2 || true
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
for w in "$@"; do
  case $w in
    tests) timeout 900 python -m pytest tests -m "gpu and not slow" -q -x -p no:cacheprovider 2>&1 | tail -40 > gpurun_out/${TAG}_tests.log ;;
    slow) timeout 1500 python -m pytest tests -m "gpu and slow" -q -x -s -p no:cacheprovider 2>&1 | tail -40 > gpurun_out/${TAG}_slow.log ;;
  esac
done
for c in $CFGS; do
  timeout 600 python bench.py --config $c --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_bench_$c.log 2>&1
done
ls gpurun_out | grep ${TAG}_
