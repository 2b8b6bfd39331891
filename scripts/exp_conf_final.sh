set -u
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -1
for c in c3 c2; do timeout 600 python bench.py --config $c --steps 10 --no-e2e --no-cpu-baseline 2>/dev/null | grep "^{" | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(\"$c\", j['ms_per_step'], j['breakdown_ms'], j['roofline']['frac'])"; done
