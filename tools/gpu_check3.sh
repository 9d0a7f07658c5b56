#!/bin/bash
set -u
OUT=gpurun_out/${1:-check3}; mkdir -p $OUT
timeout 1200 python -m pytest tests -x -q -m gpu > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest.log
B="python bench.py --no-cpu-baseline --no-e2e --no-est --no-ttft"
for rep in 1 2 3; do
  timeout 300 $B 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);c=j['ctx_131072'];print('32k',j['ms_per_step'],j['stage_ms'],' 128k',c['value'],c['stage_ms'])"
done
SAN_TESTS="tests/test_gpu_block_screen.py tests/test_gpu_api.py tests/test_gpu_layers.py" SAN_K="screen or numpy or golden or error or layer" TOOLS="initcheck" bash tools/gpu_sanitize.sh > $OUT/san.txt 2>&1
cp gpurun_out/san_initcheck.log $OUT/ 2>/dev/null; cat $OUT/san.txt
