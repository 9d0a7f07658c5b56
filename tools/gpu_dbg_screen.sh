OUT=gpurun_out/dbg11; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_block_screen.py -x -q > $OUT/pytest_screen.log 2>&1; echo "screen tests rc=$?"; tail -4 $OUT/pytest_screen.log
python tools/screen_debug.py 32768 8 1 25 | tail -3
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/l.csv python tools/screen_debug.py 32768 8 1 25 > /dev/null 2>&1
python tools/launch_summary.py $OUT/l.csv | grep -v "at::"
B="python bench.py --no-cpu-baseline --no-e2e --no-est --no-ttft"
for rep in 1 2; do
for S in 1 0; do
  SA_BLOCK_SCREEN=$S timeout 300 $B 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);c=j['ctx_131072'];print('screen=$S 32k',j['ms_per_step'],' 128k',c['value'],c['stage_ms'])"
done
done
