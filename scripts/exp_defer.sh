set -u
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
SB_LIB_PATH=$PWD/build/lib_defer.so timeout 1200 python -m pytest tests/test_gpu_parity.py -m "gpu and not slow" -x -q -p no:cacheprovider 2>&1 | tail -1
bash scripts/exp_ab.sh defer
