set -u
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r4m_build.log 2>&1
timeout 1800 python -m pytest tests -m "gpu and not slow" -q -p no:cacheprovider > gpurun_out/r4m_tests.log 2>&1
tail -3 gpurun_out/r4m_tests.log
for c in c4 c2; do timeout 600 python bench.py --config $c --steps 10 --no-e2e --no-cpu-baseline | grep "^{" | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(\"$c\", j[\"ms_per_step\"], j[\"breakdown_ms\"][\"select\"], j[\"roofline\"][\"frac\"])"; done
