set -u
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r4c_build.log 2>&1
export SB_LIB_PATH=$PWD/build/lib_trace.so
timeout 300 python scripts/sv_trace.py c2 > gpurun_out/r4c_sv_c2.txt 2>&1
timeout 300 python scripts/sv_trace.py c1one > gpurun_out/r4c_sv_c1.txt 2>&1
