set -u
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r3f_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -4 > gpurun_out/r3f_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3f_smoke.log 2>&1
timeout 900 python bench.py --record gpurun_out/r3f_runs.jsonl > gpurun_out/r3f_bench_c4.log 2>&1
for c in c1 c2 c3 c5; do timeout 600 python bench.py --config $c --steps 20 --no-e2e --record gpurun_out/r3f_runs.jsonl > gpurun_out/r3f_bench_$c.log 2>&1; done
for c in spawn kv tree hrad; do timeout 300 python bench.py --config $c --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/r3f_bench_$c.log 2>&1; done
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r3f_bench_ref.log 2>&1
timeout 600 python scripts/shard_sweep.py c5 > gpurun_out/r3f_shard_sweep.txt 2>&1
