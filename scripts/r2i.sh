set -u
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2i_build.log 2>&1
bash scripts/r2_variants.sh r2i c2 "default flow" > gpurun_out/r2i_variants_c2.txt 2>&1
bash scripts/r2_variants.sh r2i c1 "default flow fstep" > gpurun_out/r2i_variants_c1.txt 2>&1
