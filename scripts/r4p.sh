set -u
export PYTHONUNBUFFERED=1
export SB_LIB_PATH=$PWD/build/lib_trace.so
SB_ASTEP=0 timeout 300 python scripts/step_trace.py c2fixed > gpurun_out/r4p_c2fixed.txt 2>&1
