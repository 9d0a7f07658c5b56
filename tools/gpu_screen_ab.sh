#!/bin/bash
# Block screen: parity tests, then A/B of the layer (SA_BLOCK_SCREEN=1 / 0) at 32K and 128K.
set -u
OUT=gpurun_out/${1:-screen}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_block_screen.py -x -q > $OUT/pytest_screen.log 2>&1; echo "screen tests rc=$?"; tail -15 $OUT/pytest_screen.log
timeout 900 python -m pytest tests -x -q -m gpu -k "block or prefill or fullsize or golden" > $OUT/pytest_block.log 2>&1; echo "block tests rc=$?"; tail -3 $OUT/pytest_block.log
B="python bench.py --no-cpu-baseline --no-e2e --no-est --no-ttft"
for rep in 1 2; do
for S in 1 0; do
  SA_BLOCK_SCREEN=$S timeout 300 $B 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);c=j['ctx_131072'];print('screen=$S 32k',j['ms_per_step'],j['stage_ms'],' 128k',c['value'],c['stage_ms'])"
done
done
timeout 300 nsys --version >/dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-128k --no-est --no-ttft > /dev/null 2>&1; echo "ncu rc=$?"
python tools/launch_summary.py $OUT/launches.csv | head -30
