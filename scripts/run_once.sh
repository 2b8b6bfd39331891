set -u
export PYTHONUNBUFFERED=1
T=${TAG:-x}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 900 python -m pytest tests -m "gpu and not slow" -q -x 2>&1 | tail -30 > gpurun_out/${T}_tests.log
for c in c4 c1 c2 c3 c5; do timeout 600 python bench.py --config $c --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/${T}_bench_$c.log 2>&1; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_select" -s 3 -c 1 -o gpurun_out/${T}_select_c4 python bench.py --config c4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_ncu_select.log 2>&1
