#!/bin/bash
set -u
OUT=gpurun_out/san2; mkdir -p $OUT
timeout 900 python -m pytest tests -x -q -m gpu -k "kernels or api or fullsize" > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest.log
SAN_TESTS="tests/test_gpu_kernels.py tests/test_gpu_api.py" SAN_K="attention or sparse or prefill or golden" TOOLS="synccheck racecheck memcheck" bash tools/gpu_sanitize.sh > $OUT/san.txt 2>&1
cp gpurun_out/san_*.log $OUT/ 2>/dev/null; cat $OUT/san.txt
