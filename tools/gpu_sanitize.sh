# compute-sanitizer over tools/sanitize_smoke.py (memcheck, racecheck, synccheck) -> gpurun_out/sanitizers.md
set -u
OUT=gpurun_out; mkdir -p $OUT
python tools/sanitize_smoke.py > $OUT/san_plain.log 2>&1; tail -2 $OUT/san_plain.log
for tool in memcheck synccheck racecheck; do
  timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_smoke.py > $OUT/san_$tool.log 2>&1
  echo "== $tool"; tail -4 $OUT/san_$tool.log
done
