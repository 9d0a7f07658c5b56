#!/bin/bash
# VS estimator A/B over env settings: all-VS layers at 32K and 128K, ncu launch list.
set -u
OUT=gpurun_out/${1:-estab}; shift
mkdir -p $OUT
for ENV in "$@"; do
  for C in 32768 131072; do
    env $ENV timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -k regex:"topk|vs_estimator|diag_add|units" -c 12 --csv --log-file $OUT/l_${C}.csv \
      python bench.py --ctx $C --pattern vs:$((C*3/64)):$((C*3/64)) --steps 2 --warmup 2 --no-e2e --no-cpu-baseline > /dev/null 2>&1
    echo "== $ENV $C"; python tools/launch_summary.py $OUT/l_$C.csv | grep -v units
  done
done
