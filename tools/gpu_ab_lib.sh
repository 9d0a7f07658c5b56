#!/bin/bash
# same-box A/B of two builds: the product .so vs paper_2412_06198_b200/$1 (default _sa_b200_prev.so)
set -u
ALT=${1:-_sa_b200_prev.so}
B="python bench.py --no-cpu-baseline --no-e2e --no-est --no-ttft --no-128k"
for rep in 1 2 3; do
for L in _sa_b200.so $ALT; do
  for P in "" "--pattern vs:1536:1536"; do
    SA_B200_LIB=paper_2412_06198_b200/$L timeout 300 $B $P 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);print('$L $P', j['ms_per_step'], j['stage_ms']['attention'])"
  done
done
done
