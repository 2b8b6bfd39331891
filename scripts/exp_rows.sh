set -u
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in r20e2 r24 r24e2 r28e2; do SB_LIB_PATH=$PWD/build/lib_$v.so timeout 900 python -m pytest tests/test_gpu_parity.py -m "gpu and not slow" -x -q -p no:cacheprovider -k "two_calls or verify_select or three_calls" 2>&1 | tail -1; done
for r in 1 2; do
  for v in default r20e2 r24 r24e2 r28e2; do
    if [ "$v" = default ]; then unset SB_LIB_PATH; else export SB_LIB_PATH=$PWD/build/lib_$v.so; fi
    timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-clocks 2>/dev/null | grep "^{" | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(\"$v c4\", j['ms_per_step'], j['breakdown_ms']['verify'])"
    timeout 600 python bench.py --config c3 --steps 10 --no-e2e --no-cpu-baseline --no-clocks 2>/dev/null | grep "^{" | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(\"$v c3\", j['ms_per_step'], j['breakdown_ms']['verify'])"
  done
done
