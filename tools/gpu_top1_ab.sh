#!/bin/bash
# k_b = 1 block index: two-pass fp16 top-1 (SA_BLOCK_SCREEN=1) vs the default split-bf16 GEMM:
# parity tests, same-box layer timings at 32K / 128K, launch list of the block kernels.
set -u
OUT=gpurun_out/${1:-top1}
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_block_screen.py tests/test_gpu_fullsize.py tests/test_gpu_kernels.py -x -q \
    > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest.log
B="python bench.py --no-cpu-baseline --no-e2e --no-est --no-ttft --no-c5"
for rep in 1 2; do
for E in "SA_BLOCK_SCREEN=0" "SA_BLOCK_SCREEN=1"; do
  env $E timeout 600 $B 2>>$OUT/bench.err | python -c "
import json,sys;j=json.load(sys.stdin);c=j['ctx_131072']
print('$E', j['ms_per_step'], j['stage_ms'], '| 128K', c['value'], c['stage_ms'])"
done
done
SA_BLOCK_SCREEN=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"block_|key_f16" --csv \
    --log-file $OUT/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-est \
    --no-ttft --no-c5 --no-128k > $OUT/ncu.log 2>&1; echo "ncu rc=$?"
python tools/launch_summary.py $OUT/launches.csv 2>/dev/null | head -20
