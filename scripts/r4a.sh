set -u
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r4a_build.log 2>&1
for c in c1 c2; do timeout 300 python bench.py --config $c --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/r4a_bench_$c.log 2>&1; done
export SB_LIB_PATH=$PWD/build/lib_trace.so
timeout 300 python scripts/astep_trace.py c2 > gpurun_out/r4a_astep_c2.txt 2>&1
timeout 300 python scripts/step_trace.py c1one > gpurun_out/r4a_c1one.txt 2>&1
