set -u
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in default fused astep default fused astep; do
  case $v in default) unset SB_FUSED_STEP; unset SB_ASTEP;; fused) export SB_FUSED_STEP=1; unset SB_ASTEP;; astep) unset SB_FUSED_STEP; export SB_ASTEP=1;; esac
  timeout 300 python bench.py --config c1 --steps 10 --no-e2e --no-cpu-baseline 2>/dev/null | grep "^{" | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(\"$v\", j[\"ms_per_step\"], j.get(\"per_round_latency_us\"))"
done
