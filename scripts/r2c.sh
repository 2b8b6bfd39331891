set -u
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2c_build.log 2>&1
timeout 1500 python -m pytest tests -m "gpu and slow" -q -s -p no:cacheprovider 2>&1 | grep -v "^\s*$" | tail -30 > gpurun_out/r2c_slow.log
bash scripts/r2_variants.sh r2c c4 "default noexp poly4 poly2 poly1" parity > gpurun_out/r2c_variants.txt 2>&1
timeout 600 python bench.py --config c2 --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/r2c_c2_default.log 2>&1
