set -u
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spawn -s 3 -c 1 -o gpurun_out/r4k_spawn \
  python bench.py --config spawn --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > gpurun_out/r4k_ncu_spawn.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tree -s 6 -c 2 -o gpurun_out/r4k_tree \
  python bench.py --config tree --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > gpurun_out/r4k_ncu_tree.log 2>&1
