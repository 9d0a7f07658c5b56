#!/bin/bash
# One gpurun call: GPU parity tests, the default bench line (32K headline with
# the 128K / estimator / TTFT sub-records and the CPU baseline), the reference
# arm, the ncu launch list of the bench command and `ncu --set full` captures
# of the attention kernel and the estimator kernels.
#   gpurun --timeout 3000 -- bash tools/gpu_full.sh [tag]
set -u
TAG=${1:-r02}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu.txt 2>&1
cp -f MEASURED_PEAKS.json $OUT/ 2>/dev/null
timeout 1200 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-128k --no-est --no-ttft --no-c5"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 2 -c 1 \
    -o $OUT/attn $CMD > $OUT/ncu_attn.log 2>&1; echo "ncu attn rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"select_kernel|vs_estimator|block_pool|block_score|topk|build_tiles|order_work|scan_fill" -s 18 -c 12 \
    -o $OUT/est $CMD > $OUT/ncu_est.log 2>&1; echo "ncu est rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:vs_estimator -s 3 -c 1 \
    -o $OUT/vs_est_131072 python tools/est_chain.py 131072 > $OUT/ncu_vs.log 2>&1; echo "ncu vs rc=$?"
ls -la $OUT
