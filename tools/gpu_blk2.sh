#!/bin/bash
# block estimator change check: parity tests, bench stage times, launch list
set -u
OUT=gpurun_out/${1:-blk2}
mkdir -p $OUT
timeout 600 python -m pytest tests -x -q -m gpu > $OUT/pytest.log 2>&1; rc=$?
echo "pytest rc=$rc"; tail -3 $OUT/pytest.log
[ $rc -ne 0 ] && exit 1
for rep in 1 2; do
  SA_OVERLAP_EST=0 timeout 200 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);print('serial 32k',j['stage_ms'],j['ms_per_step'])"
  timeout 200 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);print('32k',j['ms_per_step'])"
done
SA_OVERLAP_EST=0 timeout 300 python bench.py --ctx 131072 --steps 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);print('serial 128k',j['stage_ms'],j['ms_per_step'])"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"block" -c 20 --csv --log-file $OUT/l.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py $OUT/l.csv
