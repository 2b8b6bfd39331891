set -u
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_next.py -m gpu -x -q -p no:cacheprovider -k spawn 2>&1 | tail -2
for r in 1 2; do timeout 300 python bench.py --config spawn --steps 20 --no-e2e --no-cpu-baseline | grep "^{" | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('spawn', j['ms_per_step'], j['roofline']['frac'])"; done
