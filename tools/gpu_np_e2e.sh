OUT=gpurun_out/npe2e; mkdir -p $OUT
timeout 900 python -m pytest tests -x -q -m gpu -k "api or error or decode or golden or fullsize" > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest.log
timeout 600 python bench.py --no-cpu-baseline --no-128k --no-est --no-ttft > $OUT/bench.json 2>$OUT/bench.err; python -c "import json;j=json.load(open('$OUT/bench.json'));print(j['value'],j['e2e']['value'],j['e2e_numpy_f32'])"
