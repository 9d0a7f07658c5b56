#!/bin/bash
# session-3 randomized sweeps through the public API (the numpy float32 path, the
# fused selector, the decode cache adopted from the numpy staging copies)
set -u
OUT=gpurun_out/${1:-sweeps}; mkdir -p $OUT
timeout 1500 python tools/parity_sweep.py --api-mix --cases 160 --seed 91 --max-n 8000 > $OUT/parity_sweep_mix_s91.jsonl 2> $OUT/parity.err; echo "parity rc=$?"
tail -2 $OUT/parity_sweep_mix_s91.jsonl | cut -c1-400
timeout 1200 python tools/decode_sweep.py --cases 80 --seed 92 > $OUT/decode_sweep_s92.jsonl 2> $OUT/decode.err; echo "decode rc=$?"
tail -2 $OUT/decode_sweep_s92.jsonl | cut -c1-400
