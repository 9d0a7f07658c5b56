#!/bin/bash
# Lab batch 2: top-k parity tests + timing (rank step distributed), host copy primitives.
set -u
OUT=gpurun_out/${1:-lab2}
mkdir -p $OUT
timeout 600 python -m pytest tests -x -q -m gpu -k "topk or vs or estimator" > $OUT/pytest_topk.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_topk.log
for C in 1 0 2; do
  SA_TOPK_CLUSTER=$C timeout 300 python tools/topk_lab.py 32768 65536 131072 > $OUT/topk_lab_c$C.txt 2>&1
  grep median $OUT/topk_lab_c$C.txt | sed "s/^/cl=$C /"
done
timeout 300 python tools/e2e_lab.py > $OUT/e2e_lab.txt 2>&1; cat $OUT/e2e_lab.txt
