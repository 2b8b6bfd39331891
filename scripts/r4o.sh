set -u
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
export SB_ASTEP=1
for v in default nored nomath nomathred default nored; do
  if [ "$v" = default ]; then unset SB_LIB_PATH; else export SB_LIB_PATH=$PWD/build/lib_$v.so; fi
  echo -n "$v: "; timeout 300 python scripts/astep_fixed.py 64 2>&1 | tail -1
done
unset SB_LIB_PATH
SB_ASTEP=0 timeout 300 python scripts/astep_fixed.py 64 2>&1 | tail -1
