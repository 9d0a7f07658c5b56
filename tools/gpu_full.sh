#!/bin/bash
# One gpurun call: GPU parity tests, bench lines (32K with the CPU baseline, 128K),
# the ncu launch list of the bench command and `ncu --set full` captures of the
# attention kernel and the estimator kernels.
#   gpurun --timeout 2400 -- bash tools/gpu_full.sh [tag]
set -u
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu.txt 2>&1
cp -f MEASURED_PEAKS.json $OUT/ 2>/dev/null
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
cat $OUT/bench.json
timeout 600 python bench.py --ctx 131072 --steps 5 --no-cpu-baseline > $OUT/bench_128k.json 2> $OUT/bench_128k.err; echo "bench128k rc=$?"
cat $OUT/bench_128k.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref rc=$?"
cat $OUT/bench_ref.json
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 2 -c 1 \
    -o $OUT/attn $CMD > $OUT/ncu_attn.log 2>&1; echo "ncu attn rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"select_kernel|tail_kernel|block_pool|block_score|topk_rows|diag_combine|build_tiles|order_work" -s 16 -c 12 \
    -o $OUT/est $CMD > $OUT/ncu_est.log 2>&1; echo "ncu est rc=$?"
ls -la $OUT
