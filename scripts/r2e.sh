set -u
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2e_build.log 2>&1
timeout 900 python -m pytest tests -m "gpu and not slow" -q -x -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/r2e_tests.log
bash scripts/r2_variants.sh r2e c4 "default base" > gpurun_out/r2e_variants_c4.txt 2>&1
bash scripts/r2_variants.sh r2e c2 "default base" > gpurun_out/r2e_variants_c2.txt 2>&1
bash scripts/r2_variants.sh r2e c3 "default base" > gpurun_out/r2e_variants_c3.txt 2>&1
timeout 1500 python -m pytest tests -m "gpu and slow" -q -s -p no:cacheprovider 2>&1 | grep -v "^\s*$" | tail -12 > gpurun_out/r2e_slow.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rows_tma" -s 3 -c 1 -o gpurun_out/r2e_c4_rows \
    python bench.py --config c4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > gpurun_out/r2e_ncu_rows.log 2>&1
