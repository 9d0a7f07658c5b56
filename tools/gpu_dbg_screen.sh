OUT=gpurun_out/dbg10; mkdir -p $OUT
ncu --set full --import-source on --clock-control none -k regex:"block_refine|block_rescan" -s 2 -c 2 -o $OUT/rr python tools/screen_debug.py 32768 8 1 25 > $OUT/ncu.log 2>&1; echo ncu rc=$?
