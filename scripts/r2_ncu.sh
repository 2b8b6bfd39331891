#!/bin/bash
# ncu launch list + full captures for one config.  usage: scripts/r2_ncu.sh TAG CONFIG "kregex1 kregex2" [extra bench args]
set -u
TAG=$1; CFG=$2; KS=${3:-"k_rows_tma"}; shift 3 || true
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_${CFG}.csv \
  python bench.py --config $CFG --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph "$@" > gpurun_out/${TAG}_launch_run.log 2>&1
for k in $KS; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 6 -c 1 -o gpurun_out/${TAG}_${CFG}_${k} \
    python bench.py --config $CFG --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph "$@" > gpurun_out/${TAG}_ncu_${k}.log 2>&1
done
ls gpurun_out | grep ${TAG}_
