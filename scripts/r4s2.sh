set -u
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r4s2_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "vocabulary_parts or astep or adaptive" > gpurun_out/r4s2_tests.log 2>&1
tail -3 gpurun_out/r4s2_tests.log
for v in 0 1 0 1; do SB_ASTEP=$v timeout 300 python bench.py --config c1 --steps 10 --no-e2e --no-cpu-baseline 2>/dev/null | grep "^{" | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(\"astep=$v\", j[\"ms_per_step\"], j.get(\"per_round_latency_us\"))"; done
for s in 2 4 8; do SB_ASTEP=1 SB_ASTEP_SPLIT=$s timeout 300 python bench.py --config c1 --steps 10 --no-e2e --no-cpu-baseline 2>/dev/null | grep "^{" | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(\"split=$s\", j.get(\"per_round_latency_us\"))"; done
