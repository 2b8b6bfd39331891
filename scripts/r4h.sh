set -u
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
export SB_LIB_PATH=$PWD/build/lib_trace.so
timeout 300 python scripts/astep_trace.py c2 > gpurun_out/r4h_astep_c2.txt 2>&1
