#!/bin/bash
# A/B sweep of environment knobs on bench lines.  usage: scripts/r2_sweep.sh TAG "c2 c1" "ENV1=.. ;ENV2=..;"
set -u
TAG=$1; CFGS=$2; VARS=$3
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
IFS=';' read -ra VA <<< "$VARS"
for c in $CFGS; do
  for v in "${VA[@]}"; do
    name=$(echo "$v" | tr -c 'A-Za-z0-9_=' '_')
    env $v timeout 600 python bench.py --config $c --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_${c}_${name}.log 2>&1
    python - "$c" "$v" gpurun_out/${TAG}_${c}_${name}.log >> gpurun_out/${TAG}_summary.txt <<'PY'
import json,sys
c,v,f=sys.argv[1:]
try:
    l=[x for x in open(f) if x.startswith('{')][-1]; j=json.loads(l)
    print(c, repr(v), j['ms_per_step'], 'frac', j['logit_frac_of_peak'], 'bd', {k:v for k,v in j['breakdown_ms'].items() if k!='source'}, 'lat', j.get('per_round_latency_us'))
except Exception as e: print(c, repr(v), 'FAILED', e)
PY
  done
done
cat gpurun_out/${TAG}_summary.txt
