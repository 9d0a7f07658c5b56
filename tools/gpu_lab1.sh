#!/bin/bash
# Lab batch: attention phase profiles, top-k timing + sample rows, ncu of the 128K top-k.
set -u
OUT=gpurun_out/${1:-lab1}
mkdir -p $OUT
make prof > $OUT/make_prof.log 2>&1 || tail -20 $OUT/make_prof.log
for P in "" "--pattern vs:1638:1638" "--pattern block:8:1" "--mode dense"; do
  echo "== attn_prof $P" >> $OUT/attn_prof.txt
  SA_B200_LIB=paper_2412_06198_b200/_sa_b200_prof.so timeout 300 python tools/attn_prof.py $P >> $OUT/attn_prof.txt 2>&1
done
timeout 300 python tools/topk_lab.py 32768 65536 131072 --save $OUT/topk_rows.npz > $OUT/topk_lab.txt 2>&1
cat $OUT/topk_lab.txt
SA_TOPK_CLUSTER=2 timeout 300 python tools/topk_lab.py 32768 131072 > $OUT/topk_lab_cl2.txt 2>&1
SA_TOPK_CLUSTER=0 timeout 300 python tools/topk_lab.py 32768 131072 > $OUT/topk_lab_cl0.txt 2>&1
grep median $OUT/topk_lab_cl*.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:topk -s 1 -c 1 \
    -o $OUT/topk_131072 python tools/topk_lab.py 131072 --reps 1 > $OUT/ncu_topk.log 2>&1; echo "ncu topk rc=$?"
