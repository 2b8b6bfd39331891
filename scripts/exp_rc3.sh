set -u
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -1
for r in 1 2; do
  for v in default head; do
    if [ "$v" = default ]; then unset SB_LIB_PATH; else export SB_LIB_PATH=$PWD/build/lib_$v.so; fi
    for c in c3 c4; do timeout 600 python bench.py --config $c --steps 10 --no-e2e --no-cpu-baseline --no-clocks 2>/dev/null | grep "^{" | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(\"$v $c\", j['ms_per_step'], j['breakdown_ms']['verify_reusing_confidence_rows'], j['breakdown_ms']['verify'])"; done
  done
done
