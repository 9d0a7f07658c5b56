#!/bin/bash
# VS estimator timeline at 128K / 32K for several MUFU / FMA-pipe exp splits
for P in "0,0" "2,0" "3,0" "4,0" "3,2"; do
  echo "== SA_VS_POLY=$P"
  SA_VS_POLY=$P timeout 120 python tools/vs_trace.py 131072 | head -3
  SA_VS_POLY=$P timeout 120 python tools/vs_trace.py 32768 | head -2
done
