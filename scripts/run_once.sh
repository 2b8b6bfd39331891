set -u
export PYTHONUNBUFFERED=1
T=${TAG:-x}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 900 python -m pytest tests -m "gpu and not slow" -q -x 2>&1 | tail -2 > gpurun_out/${T}_tests.log
for r in 1 2; do for v in A B; do
  if [ $v = A ]; then L="$PWD/build/libsb_head.so"; else L=""; fi
  for c in c4 c2 c1; do SB_LIB_PATH=$L timeout 600 python bench.py --config $c --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/${T}_r${r}_${v}_$c.log 2>&1; done
done; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rows" -s 3 -c 1 -o gpurun_out/${T}_rows_c4 python bench.py --config c4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
