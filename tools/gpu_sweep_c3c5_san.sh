#!/bin/bash
# Session-3 evidence: C3 / C5 sweep with the current build, sanitizers over the
# new kernels (block screen, fp32<->bf16 staging through the numpy prefill).
set -u
OUT=gpurun_out/${1:-sweep3}; mkdir -p $OUT
timeout 1500 python tools/sweep.py --out $OUT/sweep.json > $OUT/sweep.log 2>&1; echo "sweep rc=$?"; tail -c 1500 $OUT/sweep.log
SAN_TESTS="tests/test_gpu_block_screen.py tests/test_gpu_api.py" SAN_K="screen or numpy or golden or error" TOOLS="memcheck initcheck" bash tools/gpu_sanitize.sh > $OUT/san.txt 2>&1
cp gpurun_out/san_*.log $OUT/ 2>/dev/null
cat $OUT/san.txt
