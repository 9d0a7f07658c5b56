#!/bin/bash
set -u
OUT=gpurun_out/${1:-lab3}
mkdir -p $OUT
for C in 1 0; do
  SA_TOPK_CLUSTER=$C timeout 300 python tools/topk_lab.py 32768 131072 --trace > $OUT/topk_trace_c$C.txt 2>&1
  sed "s/^/cl=$C /" $OUT/topk_trace_c$C.txt | grep -v "row "
done
