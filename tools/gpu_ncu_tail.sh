#!/bin/bash
# ncu --set full of tail_kernel<2> (all-VS 128K) with source attribution
set -u
OUT=gpurun_out/${1:-ncutail}
mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"tail_kernel" -s 3 -c 1 \
  -o $OUT/tail2 python bench.py --ctx 131072 --pattern vs:6144:6144 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ncu.log 2>&1
echo "rc=$?"; tail -3 $OUT/ncu.log
