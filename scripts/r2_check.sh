#!/bin/bash
# Round-2 GPU session: build, GPU tests (incl. slow full-size parity), smoke.
set -u
TAG=${1:-r2}
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -s -p no:cacheprovider 2>&1 | tail -60 > gpurun_out/${TAG}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
ls gpurun_out | grep ${TAG}
