#!/bin/bash
# Env-variable A/B: parity tests with the B setting, then bench lines for A and B.
#   gpurun -- env A="SA_X=1" B="SA_X=2" bash tools/gpu_env_ab.sh tag
set -u
OUT=gpurun_out/${1:-envab}
mkdir -p $OUT
A=${A:-}
B=${B:-}
env $B timeout 300 python -m pytest tests -x -q -m gpu > $OUT/pytest_b.log 2>&1; rc=$?
echo "B tests rc=$rc"; tail -15 $OUT/pytest_b.log
if [ $rc -ne 0 ]; then exit 1; fi
for rep in 1 2; do
  for V in "$A" "$B"; do
    env $V timeout 200 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);print('[$V] auto',j['stage_ms']['attention'],j['ms_per_step'],j['roofline']['achieved'])"
    env $V timeout 200 python bench.py --pattern vs:1536:1536 --steps 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);print('[$V] vs',j['stage_ms']['attention'],j['roofline']['achieved'])"
    env $V timeout 200 python bench.py --mode dense --steps 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);print('[$V] dense',j['stage_ms']['attention'],j['roofline']['achieved'])"
  done
done
