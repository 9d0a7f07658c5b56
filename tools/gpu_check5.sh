#!/bin/bash
set -u
OUT=gpurun_out/${1:-check5}; mkdir -p $OUT
timeout 1200 python -m pytest tests -x -q -m gpu > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest.log
B="python bench.py --no-cpu-baseline --no-e2e --no-est --no-ttft"
for rep in 1 2 3; do
  timeout 300 $B 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);c=j['ctx_131072'];print('32k',j['ms_per_step'],j['stage_ms']['attention'],' 128k',c['value'],c['stage_ms']['attention'])"
done
for P in "--pattern vs:1536:1536" "--pattern block:8:1" "--mode dense"; do
  timeout 300 $B --no-128k $P 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);print('$P', j['ms_per_step'], j['stage_ms']['attention'])"
done
SAN_TESTS="tests/test_gpu_kernels.py tests/test_gpu_api.py" SAN_K="attention or sparse or prefill or golden" TOOLS="synccheck racecheck" bash tools/gpu_sanitize.sh > $OUT/san.txt 2>&1
cp gpurun_out/san_*.log $OUT/ 2>/dev/null; cat $OUT/san.txt
