set -u
export PYTHONUNBUFFERED=1
T=${TAG:-x}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
for S in 18 12 9 6 4; do SB_HRAD_SPLITS=$S timeout 300 python bench.py --config hrad --steps 30 --no-cpu-baseline > gpurun_out/${T}_S$S.log 2>&1; done
for S in 16 8 4; do SB_HRAD_SPLITS=$S timeout 300 python bench.py --config hrad --hrad-batch 256 --steps 30 --no-cpu-baseline > gpurun_out/${T}_b256_S$S.log 2>&1; done
timeout 300 python bench.py --config hrad --hrad-batch 256 --steps 30 --no-cpu-baseline > gpurun_out/${T}_b256_def.log 2>&1
