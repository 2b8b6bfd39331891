#!/bin/bash
python -m paper_2506_01979_b200.build --out paper_2506_01979_b200/libspecbranch_trace.so -- -DSB_FLOW_TRACE > gpurun_out/trace_build.log 2>&1
for a in "c2" "c2 adaptive" "c1one"; do
  SB_LIB_PATH=paper_2506_01979_b200/libspecbranch_trace.so timeout 300 python scripts/flow_trace.py $a >> gpurun_out/$1_trace.txt 2>&1
done
cat gpurun_out/$1_trace.txt
