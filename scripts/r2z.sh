set -u
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2z_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -4 > gpurun_out/r2z_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2z_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r2z_bench_default.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r2z_bench_ref.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(plan|rows|select|conf|astep)" --csv --log-file gpurun_out/r2z_launches_c4.csv python bench.py --config c4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_rows_tma" -s 3 -c 1 -o gpurun_out/r2z_c4_rows python bench.py --config c4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_select_tma" -s 3 -c 1 -o gpurun_out/r2z_c4_select python bench.py --config c4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > /dev/null 2>&1
