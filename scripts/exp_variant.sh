set -u
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in 1 2; do
  for v in def 2 3 0; do
    if [ "$v" = def ]; then unset SB_ROWS_VARIANT; else export SB_ROWS_VARIANT=$v; fi
    for c in c5 c1; do timeout 600 python bench.py --config $c --steps 10 --no-e2e --no-cpu-baseline --no-clocks 2>/dev/null | grep "^{" | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(\"v=$v $c\", j['ms_per_step'], j['breakdown_ms']['verify'])"; done
  done
done
