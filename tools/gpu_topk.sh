#!/bin/bash
# top-k parity + VS estimator timing at 32K / 128K (launch list).
set -u
OUT=gpurun_out/${1:-topk}
mkdir -p $OUT
timeout 300 python -m pytest tests -x -q -m gpu -k "topk or vs or prefill" > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 $OUT/pytest.log
timeout 600 python -m pytest tests -x -q -m gpu > $OUT/pytest_all.log 2>&1; echo "pytest all rc=$?"; tail -3 $OUT/pytest_all.log
for C in 32768 131072; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"topk|tail|diag" -c 40 --csv \
    --log-file $OUT/l_$C.csv python bench.py --ctx $C --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  python tools/launch_summary.py $OUT/l_$C.csv
done
timeout 200 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);print('32k',j['stage_ms'],j['ms_per_step'])"
timeout 200 python bench.py --ctx 131072 --steps 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);print('128k',j['stage_ms'],j['ms_per_step'])"
