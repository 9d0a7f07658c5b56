#!/bin/bash
# Epilogue warpgroup (SA_ATTN_EWG=1, default) vs softmax-warp epilogue (0): GPU tests, then A/B.
set -u
OUT=gpurun_out/${1:-ewg}
mkdir -p $OUT
timeout 1200 python -m pytest tests -x -q -m gpu > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest.log
B="python bench.py --no-cpu-baseline --no-e2e --no-est --no-ttft"
for rep in 1 2; do
for E in 1 0; do
  SA_ATTN_EWG=$E timeout 300 $B 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);c=j['ctx_131072'];print('ewg=$E auto32k',j['ms_per_step'],j['stage_ms']['attention'],' 128k',c['value'],c['stage_ms']['attention'])"
  for P in "--pattern block:8:1" "--pattern vs:1536:1536" "--mode dense"; do
    SA_ATTN_EWG=$E timeout 300 $B --no-128k $P 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);print('ewg=$E $P', j['ms_per_step'], j['stage_ms']['attention'])"
  done
done
done
