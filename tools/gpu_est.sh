#!/bin/bash
# All-VS estimator timing (north-star: estimator >= 60% of HBM peak) at 32K / 128K.
set -u
OUT=gpurun_out/${1:-est}
mkdir -p $OUT
for C in 32768 131072; do
  timeout 300 python bench.py --ctx $C --pattern vs:$((C*3/64)):$((C*3/64)) --steps 3 --no-e2e --no-cpu-baseline 2>/dev/null \
    | python -c "import json,sys;j=json.load(sys.stdin);print('$C all-VS',j['stage_ms'])"
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"topk|vs_estimator|diag_add|units" -c 30 --csv --log-file $OUT/l_$C.csv \
    python bench.py --ctx $C --pattern vs:$((C*3/64)):$((C*3/64)) --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  python tools/launch_summary.py $OUT/l_$C.csv
done
