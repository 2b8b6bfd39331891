set -u
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for tool in memcheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "adaptive and astep and (c2_B64 or K8 or tiny or gamma_max or f32_mixed)" > gpurun_out/r2w_$tool.log 2>&1
  tail -5 gpurun_out/r2w_$tool.log
done
SB_ASTEP=1 timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "small_parity and astep" > gpurun_out/r2w_memcheck_plan.log 2>&1
tail -5 gpurun_out/r2w_memcheck_plan.log
