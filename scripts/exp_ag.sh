set -u
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in a16e2 a20e2 a24e2 a12; do SB_LIB_PATH=$PWD/build/lib_$v.so timeout 900 python -m pytest tests/test_gpu_parity.py -m "gpu and not slow" -x -q -p no:cacheprovider -k "astep" 2>&1 | tail -1; done
for r in 1 2; do
  for v in default a16e2 a20e2 a24e2 a12; do
    if [ "$v" = default ]; then unset SB_LIB_PATH; else export SB_LIB_PATH=$PWD/build/lib_$v.so; fi
    timeout 600 python bench.py --config c2 --steps 30 --no-e2e --no-cpu-baseline --no-clocks 2>/dev/null | grep "^{" | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(\"$v c2\", j['ms_per_step'])"
  done
done
