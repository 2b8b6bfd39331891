set -u
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
export SB_LIB_PATH=$PWD/build/lib_trace.so
timeout 300 python scripts/sv_trace.py c2 > gpurun_out/r4f_sv_c2.txt 2>&1
timeout 300 python scripts/sv_trace.py c1one > gpurun_out/r4f_sv_c1.txt 2>&1
