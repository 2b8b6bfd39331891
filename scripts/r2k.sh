set -u
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2k_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "adaptive" > gpurun_out/r2k_adaptive.log 2>&1
bash scripts/r2_variants.sh r2k c2 "default" > gpurun_out/r2k_variants_c2.txt 2>&1
SB_ASTEP=0 timeout 600 python bench.py --config c2 --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/r2k_c2_three.log 2>&1
timeout 600 python bench.py --config c3 --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/r2k_c3_astep.log 2>&1
