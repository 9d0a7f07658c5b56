#!/bin/bash
# Attention exp-split sweep: parity tests, then the 32K bench per SA_ATTN_POLY.
set -u
OUT=gpurun_out/${1:-poly}
mkdir -p $OUT
timeout 600 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu.log
for P in 0 8 4 3 2; do
  SA_ATTN_POLY=$P timeout 300 python bench.py --no-cpu-baseline --no-e2e > $OUT/bench_p$P.json 2>&1
  python -c "import json;j=json.load(open('$OUT/bench_p$P.json'));print('poly',$P,j['value'],j['stage_ms']['attention'],j['roofline']['achieved'])"
done
for P in 0 4; do
  echo "== prof poly $P"
  SA_ATTN_POLY=$P SA_B200_LIB=paper_2412_06198_b200/_sa_b200_prof.so timeout 300 python tools/attn_prof.py 2>&1 | tail -25
done
