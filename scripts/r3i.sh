set -u
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in default cw20 cw24 cw16n6; do
  if [ "$v" = default ]; then unset SB_LIB_PATH; else export SB_LIB_PATH=$PWD/build/lib_$v.so; fi
  SB_ASTEP=0 timeout 300 python bench.py --config c3 --steps 10 --no-e2e --no-cpu-baseline | grep "^{" | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(\"$v c3\", j[\"breakdown_ms\"][\"draft_confidence\"], j[\"ms_per_step\"])"
done
