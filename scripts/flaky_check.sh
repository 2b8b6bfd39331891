# Repeat the GPU suite (flakiness of the persistent / work-queue kernels) and the default bench.
set -u
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in 1 2 3; do timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -1; done
for r in 1 2; do timeout 600 python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | grep "^{" | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('c4', j['value'], j['ms_per_step'], j['roofline']['frac'], j['clocks'])"; done
