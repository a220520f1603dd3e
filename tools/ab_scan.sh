# K1x parity + config-1 bench on the current library
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_scan.py tests/test_gpu_exact.py tests/test_gpu_large_k.py tests/test_gpu_search.py tests/test_gpu_engine.py -q -x 2>&1 | tail -2
for i in 1 2; do
timeout 300 python bench.py --config c1 --no-cpu-baseline > gpurun_out/c1_$i.json 2> gpurun_out/c1_$i.err
python -c "import json; d=json.load(open('gpurun_out/c1_$i.json')); print('c1', round(d['value']), round(d['ms_per_step']*1e3,2), round(d['stages_ms']['similarity']*1e3,2), d['step_time_distribution']['median_us'], round(d['e2e']['value']))" || tail -3 gpurun_out/c1_$i.err
done
