# config-4 shape: the CTA-pair filter over fp32 keys; library variants in tools/bin/lib_<v>.so (A/B)
mkdir -p gpurun_out
cp paper_2603_17573_b200/libhsd_gpu.so tools/bin/lib_default.so
for v in ${VARIANTS:-default}; do
cp tools/bin/lib_$v.so paper_2603_17573_b200/libhsd_gpu.so
timeout 300 python bench.py --config c4 --n ${N:-2000000} --filter native --no-cpu-baseline --e2e-steps 2 > gpurun_out/c4_$v.json 2> gpurun_out/c4_$v.err
python -c "import json,sys; d=json.load(open('gpurun_out/c4_$v.json')); print('$v', d['config']['n_rows'], round(d['value']), round(d['ms_per_step'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'], round(d['roofline']['frac'],3), round(d['stages_ms']['similarity'],3))" || tail -3 gpurun_out/c4_$v.err
done
cp tools/bin/lib_default.so paper_2603_17573_b200/libhsd_gpu.so
