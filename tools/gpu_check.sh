#!/bin/bash
# Change check: attention parity tests under a tight timeout (a hung kernel
# fails fast), then the full GPU suite, then bench lines (32K auto x2, all-VS).
#   gpurun --timeout 900 -- bash tools/gpu_check.sh tag
set -u
OUT=gpurun_out/${1:-check}
mkdir -p $OUT
timeout 240 python -m pytest tests -x -q -m gpu -k "attn or prefill" > $OUT/pytest_attn.log 2>&1; rc=$?
echo "attn tests rc=$rc"; tail -25 $OUT/pytest_attn.log
if [ $rc -ne 0 ]; then exit 1; fi
timeout 600 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 $OUT/pytest_gpu.log
for rep in 1 2; do
  timeout 200 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);print('auto',j['stage_ms'],j['ms_per_step'],j['roofline']['achieved'])"
done
timeout 200 python bench.py --pattern vs:1536:1536 --steps 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);print('vs',j['stage_ms']['attention'],j['roofline']['achieved'])"
timeout 200 python bench.py --mode dense --steps 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);print('dense',j['stage_ms']['attention'],j['roofline']['achieved'])"
