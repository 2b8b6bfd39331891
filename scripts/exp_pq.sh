set -u
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/pq_build.log 2>&1
timeout 1500 python -m pytest tests -m "gpu and not slow" -x -q -p no:cacheprovider > gpurun_out/pq_tests.log 2>&1
tail -2 gpurun_out/pq_tests.log
for r in 1 2; do timeout 600 python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | grep "^{" | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('c4', j['ms_per_step'], j['breakdown_ms']['verify'], j['roofline']['frac'], j['clocks']['reasons'])"; done
for c in c3 c1 c5; do timeout 600 python bench.py --config $c --steps 10 --no-e2e --no-cpu-baseline 2>/dev/null | grep "^{" | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(\"$c\", j['ms_per_step'], j['roofline']['frac'])"; done
