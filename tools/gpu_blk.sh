#!/bin/bash
# Block estimator A/B (SA_BLOCK_FILTER=1 filter+refine vs 0 exact three-pass), parity tests first
set -u
OUT=gpurun_out/${1:-blk}
mkdir -p $OUT
timeout 300 python -m pytest tests -x -q -m gpu -k "block or prefill or golden or fullsize" > $OUT/pytest.log 2>&1; rc=$?
echo "pytest rc=$rc"; tail -15 $OUT/pytest.log
[ $rc -ne 0 ] && exit 1
for rep in 1 2; do
  for F in 1 0; do
    SA_BLOCK_FILTER=$F timeout 200 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);print('filter=$F 32k',j['stage_ms']['block_estimator'],j['ms_per_step'])"
  done
done
for F in 1 0; do
  SA_BLOCK_FILTER=$F timeout 300 python bench.py --ctx 131072 --steps 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);print('filter=$F 128k',j['stage_ms']['block_estimator'],j['ms_per_step'])"
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"block|key_norm" -c 20 --csv --log-file $OUT/l.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py $OUT/l.csv
