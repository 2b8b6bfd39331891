set -u
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for g in 1 4 5; do echo "geo $g"; SB_RW_GEO=$g timeout 600 python scripts/shard_sweep.py c5 2>&1 | tail -2; done
