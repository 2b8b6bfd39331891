set -u
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2j_build.log 2>&1
timeout 900 python bench.py --config c4 --steps 20 --record gpurun_out/r2j_runs.jsonl > gpurun_out/r2j_bench_c4.log 2>&1
for c in c1 c2 c3 c5; do timeout 600 python bench.py --config $c --steps 20 --no-e2e --record gpurun_out/r2j_runs.jsonl > gpurun_out/r2j_bench_$c.log 2>&1; done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2j_bench_ref.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2j_launches_c4.csv \
  python bench.py --config c4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rows_tma" -s 3 -c 1 -o gpurun_out/r2j_c4_rows \
    python bench.py --config c4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_select_tma" -s 3 -c 1 -o gpurun_out/r2j_c4_select \
    python bench.py --config c4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > /dev/null 2>&1
timeout 1500 python -m pytest tests -m "gpu and slow" -q -s -p no:cacheprovider 2>&1 | grep -v "^\s*$" | tail -12 > gpurun_out/r2j_slow.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2j_smoke.log 2>&1
