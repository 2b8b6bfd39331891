set -u
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in default rnored default rnored; do
  if [ "$v" = default ]; then unset SB_LIB_PATH; else export SB_LIB_PATH=$PWD/build/lib_$v.so; fi
  timeout 600 python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | grep "^{" | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(\"$v\", j['ms_per_step'], j['breakdown_ms']['verify'], j['roofline']['frac'])"
done
