#!/bin/bash
# One GPU-box pass that produces the round's evidence under gpurun_out/:
#   tests.log          pytest -m gpu
#   bench.json         default bench line (config 2), bench_{c1,c3,c4,c5,bf16}.json, bench_ref.json (--impl reference)
#   launches.csv       ncu launch list of the config-2 step (cold, serialised; --clock-control none)
#   launches_warm.csv  the same with --cache-control none
#   full_c2.ncu-rep    ncu --set full of K1 + the K2 rescoring kernel (config 2)
#   full_c4.ncu-rep    the CTA-pair filter at B = 256 (fp32, TF32) + K4
#   full_c5.ncu-rep    the CTA-pair filter at B = 683 (3 pairs per cluster, bf16)
#   full_c3.ncu-rep    K4 at config 3 (4096 episodes x 12 parameter sets)
#   full_c1.ncu-rep    K1x exact scan at config 1 (10k rows, batch 1)
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
for c in c1 c3 c4 c5 bf16; do
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
# config-5 shape: 683 queries = a cluster of 3 CTA pairs with multicast key halves (bf16 keys, 1M rows)
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:sim_pair" -s 1 -c 1 \
  -o $OUT/full_c5 python tools/bench_search.py --n 1000000 --batches 683 --dtypes bf16 --iters 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:verify" -s 2 -c 1 \
  -o $OUT/full_c3 python bench.py --config c3 --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
# config-1 shape: the K1x exact scan (10k rows, batch 1)
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:exact_scan" -s 4 -c 1 \
  -o $OUT/full_c1 python bench.py --config c1 --steps 3 --warmup 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
timeout 600 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err
# summaries on the box (gpurun returns at most 64 MiB): launch lists, full captures, DRAM traffic
cp profiles/traffic.json $OUT/traffic.json
python tools/ncu_summary.py launches $OUT/launches.csv $OUT/launches.md > /dev/null
python tools/ncu_summary.py launches $OUT/launches_warm.csv $OUT/launches_warm.md > /dev/null
python tools/ncu_summary.py full $OUT/full_c2.ncu-rep $OUT/ncu_full_c2.md --traffic $OUT/traffic.json \
  --key similarity --match sim_wide > /dev/null
python tools/ncu_summary.py full $OUT/full_c4.ncu-rep $OUT/ncu_full_c4.md --traffic $OUT/traffic.json \
  --key similarity_pair --match sim_pair > /dev/null
python tools/ncu_summary.py full $OUT/full_c5.ncu-rep $OUT/ncu_full_c5.md --traffic $OUT/traffic.json \
  --key similarity_pair_c5 --match sim_pair > /dev/null
python tools/ncu_summary.py full $OUT/full_c3.ncu-rep $OUT/ncu_full_c3.md --traffic $OUT/traffic.json \
  --key verify_c3 --match verify > /dev/null
python tools/ncu_summary.py full $OUT/full_c1.ncu-rep $OUT/ncu_full_c1.md --traffic $OUT/traffic.json \
  --key exact_scan_c1 --match exact_scan > /dev/null
# keep the config-2 report (source-level reading here); drop the rest to stay under the size cap
rm -f $OUT/full_c1.ncu-rep $OUT/full_c3.ncu-rep $OUT/full_c4.ncu-rep $OUT/full_c5.ncu-rep
ls -la $OUT
