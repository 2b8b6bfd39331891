# The N-rank launch path on a one-GPU box (ranks share cuda:0; gloo for the barrier and the
# max-over-ranks timing): bench.py --gpus 2 self-launches two ranks.
set -u
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python bench.py --gpus 2 --dist-backend gloo --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks > gpurun_out/mr_c4.log 2>&1
timeout 900 python bench.py --gpus 2 --dist-backend gloo --config c5 --mode vocab --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks > gpurun_out/mr_c5.log 2>&1
