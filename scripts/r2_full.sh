#!/bin/bash
# Round-2 GPU session: build, fast GPU tests, bench lines for all configs, slow full-size parity, smoke.
# usage: scripts/r2_full.sh TAG
set -u
TAG=${1:-r2}
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 900 python -m pytest tests -m "gpu and not slow" -q -p no:cacheprovider 2>&1 | tail -40 > gpurun_out/${TAG}_tests.log
timeout 900 python bench.py --config c4 --steps 10 > gpurun_out/${TAG}_bench_c4.log 2>&1
for c in c1 c2 c3 c5; do timeout 600 python bench.py --config $c --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_bench_$c.log 2>&1; done
timeout 1500 python -m pytest tests -m "gpu and slow" -q -s -p no:cacheprovider 2>&1 | tail -60 > gpurun_out/${TAG}_slow.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
ls gpurun_out | grep ${TAG}_
