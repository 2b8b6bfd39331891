set -u
export PYTHONUNBUFFERED=1
T=${TAG:-x}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_next.py -q -x -k hrad 2>&1 | tail -30 > gpurun_out/${T}_tests.log
for b in 2048 256 8192; do timeout 300 python bench.py --config hrad --hrad-batch $b --steps 30 --no-cpu-baseline > gpurun_out/${T}_hrad_${b}.log 2>&1; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_hrad" -s 6 -c 2 -o gpurun_out/${T}_hrad python bench.py --config hrad --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_ncu_hrad.log 2>&1
