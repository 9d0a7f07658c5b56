#!/bin/bash
# Quick GPU check: kernel parity tests + one bench line.
#   gpurun --timeout 900 -- bash tools/gpu_quick.sh tag [pytest -k expr]
set -u
TAG=${1:-quick}
K=${2:-}
OUT=gpurun_out/$TAG
mkdir -p $OUT
if [ -n "$K" ]; then
  timeout 600 python -m pytest tests -x -q -m gpu -k "$K" > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"
else
  timeout 600 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"
fi
tail -15 $OUT/pytest_gpu.log
timeout 300 python bench.py --no-cpu-baseline --no-e2e > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
cat $OUT/bench.json; tail -5 $OUT/bench.err
