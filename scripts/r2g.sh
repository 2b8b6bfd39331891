set -u
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2g_build.log 2>&1
bash scripts/r2_variants.sh r2g c4 "default nowd rv5 base" > gpurun_out/r2g_variants_c4.txt 2>&1
bash scripts/r2_variants.sh r2g c3 "default nowd rv5" > gpurun_out/r2g_variants_c3.txt 2>&1
bash scripts/r2_variants.sh r2g c2 "default nowd rv5" > gpurun_out/r2g_variants_c2.txt 2>&1
SB_ROWS_VARIANT=5 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "small" > gpurun_out/r2g_par_rv5.log 2>&1
