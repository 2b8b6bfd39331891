set -u
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py tests/test_gpu_confidence.py tests/test_gpu_shard.py tests/test_gpu_next.py -q -p no:cacheprovider -k "not full_size and not single_launch and not astep" > gpurun_out/r2x_memcheck.log 2>&1
tail -4 gpurun_out/r2x_memcheck.log
timeout 1500 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_parity.py tests/test_gpu_confidence.py -q -p no:cacheprovider -k "not full_size and not single_launch and not astep" > gpurun_out/r2x_synccheck.log 2>&1
tail -4 gpurun_out/r2x_synccheck.log
