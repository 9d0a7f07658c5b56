#!/bin/bash
# Phase-cycle profiles (prof build) for a few workloads; env passes through.
set -u
export SA_B200_LIB=paper_2412_06198_b200/_sa_b200_prof.so
for P in "" "--pattern vs:1536:1536" "--mode dense"; do
  echo "=== $P"
  timeout 200 python tools/attn_prof.py $P 2>&1 | tail -30
done
