#!/bin/bash
# ncu launch list (device time per kernel) of one bench step; summary printed.
OUT=gpurun_out/${1:-launches}
mkdir -p $OUT
shift
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline "$@" > $OUT/ncu.log 2>&1
python tools/launch_summary.py $OUT/launches.csv
