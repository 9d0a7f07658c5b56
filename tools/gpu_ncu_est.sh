#!/bin/bash
# ncu --set full of the VS estimator kernel on an all-VS layer (default 32K).
set -u
OUT=gpurun_out/${1:-ncu_est}
C=${2:-32768}
mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:vs_estimator -s 3 -c 1 \
  -o $OUT/vs_$C python bench.py --ctx $C --pattern vs:$((C*3/64)):$((C*3/64)) --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ncu.log 2>&1
echo "ncu rc=$?"; tail -3 $OUT/ncu.log
