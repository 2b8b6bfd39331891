set -u
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2r_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py tests/test_gpu_next.py -q -x -p no:cacheprovider 2>&1 | tail -3 > gpurun_out/r2r_tests.log
bash scripts/r2_variants.sh r2r c4 "default base" > gpurun_out/r2r_variants_c4.txt 2>&1
bash scripts/r2_variants.sh r2r c3 "default base" > gpurun_out/r2r_variants_c3.txt 2>&1
