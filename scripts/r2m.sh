set -u
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2m_build.log 2>&1
timeout 300 ./scripts/readbw > gpurun_out/r2m_readbw.log 2>&1
bash scripts/r2_variants.sh r2m c4 "default legacy" > gpurun_out/r2m_variants_c4.txt 2>&1
bash scripts/r2_variants.sh r2m c2 "default legacy" > gpurun_out/r2m_variants_c2.txt 2>&1
