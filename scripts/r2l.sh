set -u
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2l_build.log 2>&1
SB_LIB_PATH=$PWD/build/lib_trace.so timeout 300 python scripts/astep_trace.py c2 > gpurun_out/r2l_astep_c2.log 2>&1
bash scripts/r2_variants.sh r2l c4 "default hint" > gpurun_out/r2l_variants_c4.txt 2>&1
bash scripts/r2_variants.sh r2l c2 "default hint" > gpurun_out/r2l_variants_c2.txt 2>&1
timeout 900 python -m pytest tests -m "gpu and not slow" -q -p no:cacheprovider 2>&1 | tail -4 > gpurun_out/r2l_tests.log
