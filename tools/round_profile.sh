#!/bin/bash
# One GPU-box pass that produces the round's evidence under gpurun_out/:
#   tests.log       pytest -m gpu
#   bench.json      default bench line (config 2) + bench_c1/c3/c4/c5 lines
#   launches.csv    ncu launch list (cold, serialised; --clock-control none)
#   launches_warm.csv  the same with --cache-control none
#   full_c2.ncu-rep    ncu --set full of K1 + the K2 rescoring kernel
# Usage: gpurun --timeout 3000 -- bash tools/round_profile.sh [quick]
set -u
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $OUT/gpu.txt 2>&1
if [ "${1:-}" != "quick" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/tests.log 2>&1
  tail -3 $OUT/tests.log
fi
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
cat $OUT/bench.json
for c in c1 c3 c4 c5; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
ARGS="python bench.py --steps 3 --warmup 1 --no-cpu-baseline --e2e-steps 1"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/launches.csv $ARGS > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 60 --csv \
  --log-file $OUT/launches_warm.csv $ARGS > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:sim_wide|rescore" -s 6 -c 2 \
  -o $OUT/full_c2 $ARGS > /dev/null 2>&1
# config-4 shape (B = 256, CTA-pair filter) on a 2M-row DB to bound the replay time
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:sim_pair|verify" -s 2 -c 2 \
  -o $OUT/full_c4 python bench.py --config c4 --n 2000000 --filter native --steps 2 --warmup 1 --no-cpu-baseline \
  --e2e-steps 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:verify" -s 2 -c 1 \
  -o $OUT/full_c3 python bench.py --config c3 --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
ls -la $OUT
