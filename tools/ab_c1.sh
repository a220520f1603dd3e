# same-box A/B of the config-1 round: HEAD library (tools/bin/lib_orig.so) vs the working tree (tools/bin/lib_new.so)
for rep in 1 2; do for v in orig new; do
  cp tools/bin/lib_$v.so paper_2603_17573_b200/libhsd_gpu.so
  python tools/c1_breakdown.py 2>&1 | grep "step: full\|bench-like 200 steps  " | sed "s/^/$v /"
  timeout 300 python bench.py --config c1 --no-cpu-baseline --e2e-steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v c1', round(d['value']), round(d['ms_per_step']*1e3,2))"
done; done
cp tools/bin/lib_new.so paper_2603_17573_b200/libhsd_gpu.so
