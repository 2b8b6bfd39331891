set -u
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -q -x -p no:cacheprovider -k "rows_warp or sharded_loopback" 2>&1 | tail -5
timeout 600 python scripts/shard_sweep.py c5 2>&1 | tail -4
SB_ROWS_VARIANT=2 timeout 600 python scripts/shard_sweep.py c5 2>&1 | tail -4
