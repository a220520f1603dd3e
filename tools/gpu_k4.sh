set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_verify.py tests/test_gpu_chains.py tests/test_gpu_engine.py tests/test_gpu_hybrid.py -q -x > $OUT/k4_tests.log 2>&1; tail -3 $OUT/k4_tests.log
timeout 300 python bench.py --config c3 --no-cpu-baseline > $OUT/k4_bench_c3.json 2>$OUT/k4_bench_c3.err; tail -c 600 $OUT/k4_bench_c3.json | head -c 600; echo
timeout 300 python bench.py --no-cpu-baseline > $OUT/k4_bench_c2.json 2>&1; python -c "import json;d=json.loads(open('$OUT/k4_bench_c2.json').read().strip().splitlines()[-1]);print('c2',d['value'],d['e2e']['value'])"
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:verify" -s 2 -c 1 -o $OUT/full_c3 python bench.py --config c3 --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
python tools/ncu_summary.py full $OUT/full_c3.ncu-rep $OUT/ncu_full_c3.md --traffic $OUT/traffic_tmp.json --key verify_c3 --match verify > /dev/null 2>&1; cat $OUT/ncu_full_c3.md
