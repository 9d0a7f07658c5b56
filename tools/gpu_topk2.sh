#!/bin/bash
OUT=gpurun_out/topk2; mkdir -p $OUT
timeout 900 python -m pytest tests -x -q -m gpu -k "topk or vs or estimator or fullsize" > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest.log
for C in 1 0; do
  SA_TOPK_CLUSTER=$C timeout 300 python tools/topk_lab.py 32768 65536 131072 --trace > $OUT/topk_trace_c$C.txt 2>&1
  sed "s/^/cl=$C /" $OUT/topk_trace_c$C.txt | grep -v "row "
done
timeout 300 python tools/est_ab.py 32768 131072
