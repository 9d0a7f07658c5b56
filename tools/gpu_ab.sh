#!/bin/bash
# A/B of attention variants on one box (bench attention stage ms).
set -u
OUT=gpurun_out/${1:-ab}
mkdir -p $OUT
ROOT=$(pwd)
run() {  # name dir env...
  local name=$1; local dir=$2; shift; shift
  (cd $dir && env "$@" timeout 300 python bench.py --no-cpu-baseline --no-e2e > $ROOT/$OUT/bench_$name.json 2>&1)
  python -c "import json;j=json.load(open('$OUT/bench_$name.json'));print('$name',j['value'],j['stage_ms']['attention'],j['roofline']['achieved'])" 2>/dev/null || tail -3 $OUT/bench_$name.json
}
for v in ${VARIANTS:-old}; do run $v scratch/$v; done
