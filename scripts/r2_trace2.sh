#!/bin/bash
for mb in 3 2; do
  for a in "c2" "c1one"; do
    echo "== minblocks $mb" >> gpurun_out/$1_trace.txt
    SB_LIB_PATH=paper_2506_01979_b200/libspecbranch_trace$mb.so timeout 300 python scripts/flow_trace.py $a >> gpurun_out/$1_trace.txt 2>&1
  done
done
cat gpurun_out/$1_trace.txt
