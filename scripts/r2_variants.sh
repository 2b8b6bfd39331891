#!/bin/bash
# A/B of experiment builds (build/lib_<name>.so, SB_LIB_PATH) on one box.
# usage: scripts/r2_variants.sh TAG CONFIG "default noexp poly4 ..." [parity]
set -u
TAG=$1; CFG=$2; VARS=$3; PAR=${4:-}
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
for v in $VARS; do
  unset SB_LIB_PATH SB_ROWS_VARIANT SB_FLOW SB_FUSED_STEP
  case $v in
    default) ;;
    flow) export SB_FLOW=1 ;;
    fstep) export SB_FUSED_STEP=1 ;;
    rv*) export SB_ROWS_VARIANT=${v#rv} ;;   # geometry variant of the default library
    *) export SB_LIB_PATH=$PWD/build/lib_$v.so ;;
  esac
  for rep in 1 2; do
    timeout 600 python bench.py --config $CFG --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_${CFG}_${v}_$rep.log 2>&1
  done
  if [ -n "$PAR" ] && [ "$v" != default ] && [ "$v" != noexp ]; then
    timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "small or special or identical" > gpurun_out/${TAG}_par_${v}.log 2>&1
  fi
done
unset SB_LIB_PATH SB_ROWS_VARIANT SB_FLOW SB_FUSED_STEP
python - <<'PY'
import glob, json, re, os
tag = os.environ.get("TAG_", "")
for f in sorted(glob.glob("gpurun_out/*_*_*_[12].log")):
    try:
        line = [l for l in open(f) if l.startswith("{")][-1]
        j = json.loads(line)
        print(f, j["ms_per_step"], j["breakdown_ms"].get("verify"), j["roofline"]["frac"], j["clocks"], j.get("per_round_latency_us"))
    except Exception as e:
        print(f, "ERR", e)
PY
