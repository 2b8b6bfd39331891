# A/B of two library builds on one box: default (in-tree) vs build/lib_$1.so
set -u
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
B=${1:-head}
for r in 1 2 3; do
  for v in default $B; do
    if [ "$v" = default ]; then unset SB_LIB_PATH; else export SB_LIB_PATH=$PWD/build/lib_$v.so; fi
    timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-clocks 2>/dev/null | grep "^{" | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(\"$v c4\", j['ms_per_step'], j['breakdown_ms']['verify'])"
    for c in c1 c3; do timeout 600 python bench.py --config $c --steps 10 --no-e2e --no-cpu-baseline --no-clocks 2>/dev/null | grep "^{" | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(\"$v $c\", j['ms_per_step'], j['breakdown_ms']['verify'])"; done
  done
done
