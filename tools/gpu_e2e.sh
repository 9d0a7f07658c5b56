#!/bin/bash
# host-streamed e2e A/B over SA_STREAM_TAIL_PIECES (row pieces of the last kv group)
set -u
OUT=gpurun_out/${1:-e2e}
mkdir -p $OUT
timeout 300 python -m pytest tests -x -q -m gpu -k "host_streamed or batched or golden or prefill" > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest.log
for rep in 1 2; do
  for P in 1 2 3; do
    SA_D2H_STREAMS=$P timeout 300 python bench.py --steps 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);print('d2h_streams=$P e2e',j['e2e']['value'],'device',j['ms_per_step'])"
  done
done
for P in 1 2; do
  SA_D2H_STREAMS=$P timeout 300 python bench.py --ctx 131072 --steps 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);print('128k d2h_streams=$P e2e',j['e2e']['value'],'device',j['ms_per_step'])"
done
SA_D2H_STREAMS=2 timeout 300 python tools/e2e_timeline.py --ctx 32768 | tail -10
