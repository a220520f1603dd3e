# A/B of the config-1 step: K4 launched early (PDL under K1x) vs after the join; graph replay vs eager.
mkdir -p gpurun_out
for g in "" "--eager"; do
for v in early base; do
if [ $v = base ]; then export HSD_NO_EARLY_VERIFY=1; else unset HSD_NO_EARLY_VERIFY; fi
timeout 300 python bench.py --config c1 --no-cpu-baseline --e2e-steps 1 $g > gpurun_out/c1_$v.json 2>gpurun_out/c1_$v.err
python -c "
import json; d=json.load(open('gpurun_out/c1_$v.json')); print('$v $g', round(d['value']), round(d['ms_per_step']*1e3,2), {k: round(v, 1) for k, v in d['step_time_distribution'].items()})" || tail -3 gpurun_out/c1_$v.err
done; done
