#!/bin/bash
# compute-sanitizer passes over the small-size API / integration GPU tests
# (caching allocator off so out-of-bounds accesses inside torch's pools are seen).
set -u
mkdir -p gpurun_out
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
for TOOL in ${TOOLS:-memcheck synccheck}; do
  echo "=== $TOOL ${SAN_EXCL:-}"
  timeout ${SAN_TIMEOUT:-1200} compute-sanitizer --tool $TOOL --target-processes all --print-limit 20 ${SAN_EXCL:+--kernel-name-exclude kns=$SAN_EXCL} \
    --log-file gpurun_out/san_$TOOL.log \
    python -m pytest ${SAN_TESTS:-tests/test_gpu_api.py tests/test_integration_doc.py} -m gpu -x -q -p no:cacheprovider \
    ${SAN_K:+-k "$SAN_K"} 2>&1 | tail -3
  echo "rc=$?"; grep -c "=========" gpurun_out/san_$TOOL.log; grep -m5 "ERROR SUMMARY\|Invalid\|Race\|Barrier\|error" gpurun_out/san_$TOOL.log
done
