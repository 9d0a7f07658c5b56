#!/bin/bash
# estimator parity tests (tight timeout) + all-VS estimator timing
set -u
OUT=gpurun_out/${1:-estc}
mkdir -p $OUT
timeout 300 python -m pytest tests -x -q -m gpu > $OUT/pytest.log 2>&1; rc=$?
echo "pytest rc=$rc"; tail -8 $OUT/pytest.log
[ $rc -ne 0 ] && exit 1
bash tools/gpu_est.sh ${1:-estc}
