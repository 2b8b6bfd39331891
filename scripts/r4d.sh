set -u
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r4d_build.log 2>&1
for c in c2 c1one; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sv -s 3 -c 1 -o gpurun_out/r4d_sv_$c \
    python scripts/sv_run.py $c > gpurun_out/r4d_ncu_$c.log 2>&1
done
