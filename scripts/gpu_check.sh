#!/bin/bash
# One GPU session: parity tests, benches, ncu launch list + full capture of the top kernels.
# usage: scripts/gpu_check.sh TAG [tests|bench|ncu ...]
set -u
TAG=${1:-r}; shift
WHAT=${*:-"tests bench ncu"}
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
for w in $WHAT; do
  case $w in
    tests) timeout 900 python -m pytest tests -m "gpu and not slow" -q -x 2>&1 | tail -30 > gpurun_out/${TAG}_tests.log ;;
    slow) timeout 1200 python -m pytest tests -m "gpu and slow" -q -x -s 2>&1 | tail -40 > gpurun_out/${TAG}_slow.log ;;
    readbw) ./scripts/readbw > gpurun_out/${TAG}_readbw.log 2>&1 ;;
    ref) timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_ref.log 2>&1 ;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1 ;;
    bench) timeout 900 python bench.py --config c4 --steps 10 > gpurun_out/${TAG}_bench_c4.log 2>&1
           for c in c1 c2 c3 c5; do timeout 600 python bench.py --config $c --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_bench_$c.log 2>&1; done ;;
    ncusel) timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_select" -s 3 -c 1 -o gpurun_out/${TAG}_select_c4 python bench.py --config c4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_ncu_select.log 2>&1 ;;
    ncu) timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(plan|rows|select|conf)" --csv --log-file gpurun_out/${TAG}_launches_c4.csv python bench.py --config c4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
         timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rows" -s 3 -c 1 -o gpurun_out/${TAG}_rows_c4 python bench.py --config c4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_ncu_rows.log 2>&1
         timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_select" -s 3 -c 1 -o gpurun_out/${TAG}_select_c4 python bench.py --config c4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_ncu_select.log 2>&1 ;;
  esac
done
ls gpurun_out
