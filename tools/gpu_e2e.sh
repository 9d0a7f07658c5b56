#!/bin/bash
# host-streamed e2e A/B: output D2H by SM copy kernel vs copy-engine 2-D DMA,
# tail unit width, copy CTAs
set -u
OUT=gpurun_out/${1:-e2e}
mkdir -p $OUT
timeout 300 python -m pytest tests -x -q -m gpu -k "host_streamed or batched or golden" > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest.log
for V in "SA_D2H_SM=0 SA_STREAM_TAIL=4" "SA_D2H_SM=1 SA_STREAM_TAIL=4" "SA_D2H_SM=1 SA_STREAM_TAIL=1" "SA_D2H_SM=1 SA_STREAM_TAIL=2" "SA_D2H_SM=1 SA_STREAM_TAIL=1 SA_D2H_BLOCKS=32" "SA_D2H_SM=1 SA_STREAM_TAIL=1 SA_D2H_BLOCKS=148"; do
  for rep in 1 2; do
    env $V timeout 300 python bench.py --steps 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);print('[$V] e2e',j['e2e']['value'],'device',j['ms_per_step'])"
  done
done
for V in "SA_D2H_SM=0 SA_STREAM_TAIL=4" "SA_D2H_SM=1 SA_STREAM_TAIL=1"; do
  env $V timeout 300 python bench.py --ctx 131072 --steps 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);print('128k [$V] e2e',j['e2e']['value'],'device',j['ms_per_step'])"
done
SA_D2H_SM=1 SA_STREAM_TAIL=1 timeout 300 python tools/e2e_timeline.py --ctx 32768 | tail -12
