set -u
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m "gpu and not slow" -q -p no:cacheprovider 2>&1 | tail -3
timeout 600 python scripts/shard_sweep.py c5 > gpurun_out/r3e_shard_sweep.txt 2>&1; tail -4 gpurun_out/r3e_shard_sweep.txt
SB_ROWS_VARIANT=2 timeout 600 python scripts/shard_sweep.py c5 > gpurun_out/r3e_shard_sweep_tma.txt 2>&1; tail -4 gpurun_out/r3e_shard_sweep_tma.txt
