# Round-2 final evidence run (one box): GPU suite incl. slow full-size parity, smoke, the
# default bench line, the other configs, the reference arm, launch list + ncu captures.
set -u
export PYTHONUNBUFFERED=1
T=${1:-r4f}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -4 > gpurun_out/${T}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 900 python bench.py --record gpurun_out/${T}_runs.jsonl > gpurun_out/${T}_bench_c4.log 2>&1
for c in c1 c2 c3 c5; do timeout 600 python bench.py --config $c --steps 20 --no-e2e --record gpurun_out/${T}_runs.jsonl > gpurun_out/${T}_bench_$c.log 2>&1; done
for c in spawn kv tree hrad; do timeout 300 python bench.py --config $c --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/${T}_bench_$c.log 2>&1; done
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/${T}_bench_ref.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_c4.csv \
  -k regex:"k_(plan|rows|select|conf|astep)" python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > gpurun_out/${T}_launch_run.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rows_tma -s 6 -c 1 -o gpurun_out/${T}_c4_rows \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > gpurun_out/${T}_ncu_rows.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_astep -s 6 -c 1 -o gpurun_out/${T}_c2_astep \
  python bench.py --config c2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > gpurun_out/${T}_ncu_astep.log 2>&1
ls gpurun_out | grep "^${T}_"
