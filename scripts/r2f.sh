set -u
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2f_build.log 2>&1
timeout 900 python -m pytest tests -m "gpu and not slow" -q -p no:cacheprovider 2>&1 | tail -8 > gpurun_out/r2f_tests.log
bash scripts/r2_variants.sh r2f c4 "default base" > gpurun_out/r2f_variants_c4.txt 2>&1
bash scripts/r2_variants.sh r2f c2 "default base" > gpurun_out/r2f_variants_c2.txt 2>&1
bash scripts/r2_variants.sh r2f c3 "default base" > gpurun_out/r2f_variants_c3.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rows_tma" -s 3 -c 1 -o gpurun_out/r2f_c4_rows \
    python bench.py --config c4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > gpurun_out/r2f_ncu_rows.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rows_tma" -s 3 -c 1 -o gpurun_out/r2f_c2_rows \
    python bench.py --config c2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > gpurun_out/r2f_ncu_rows2.log 2>&1
