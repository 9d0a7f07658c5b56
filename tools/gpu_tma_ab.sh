#!/bin/bash
# TMA-store epilogue variant (_sa_b200_tma.so) vs the product build: parity tests, then A/B.
set -u
OUT=gpurun_out/${1:-tma}
mkdir -p $OUT
SA_B200_LIB=paper_2412_06198_b200/_sa_b200_tma.so timeout 1200 python -m pytest tests -x -q -m gpu -k "not multigpu and not bench" > $OUT/pytest_tma.log 2>&1; echo "pytest(tma) rc=$?"; tail -3 $OUT/pytest_tma.log
B="python bench.py --no-cpu-baseline --no-e2e --no-est --no-ttft"
for rep in 1 2; do
for L in _sa_b200_tma.so _sa_b200.so; do
  SA_B200_LIB=paper_2412_06198_b200/$L timeout 300 $B 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);c=j['ctx_131072'];print('$L auto32k',j['ms_per_step'],j['stage_ms']['attention'],' 128k',c['value'],c['stage_ms']['attention'])"
  for P in "--pattern block:8:1" "--pattern vs:1536:1536"; do
    SA_B200_LIB=paper_2412_06198_b200/$L timeout 300 $B --no-128k $P 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);print('$L $P', j['ms_per_step'], j['stage_ms']['attention'])"
  done
done
done
