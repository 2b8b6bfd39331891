set -u
export PYTHONUNBUFFERED=1
T=${TAG:-x}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 600 python -m pytest tests -m "gpu and not slow" -q -x 2>&1 | tail -30 > gpurun_out/${T}_tests.log
SB_DISABLE_TMA=1 timeout 300 python -m pytest tests/test_gpu_next.py -q -x -k spawn 2>&1 | tail -3 > gpurun_out/${T}_tests_notma.log
for c in spawn kv tree; do timeout 600 python bench.py --config $c --steps 20 > gpurun_out/${T}_bench_$c.log 2>&1; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spawn" -s 3 -c 1 -o gpurun_out/${T}_spawn python bench.py --config spawn --steps 1 --warmup 3 > gpurun_out/${T}_ncu_spawn.log 2>&1
