#!/usr/bin/env bash
# Round profile on one B200 (run under gpurun from the repo root):
#   1. ncu launch list of the bench's timed region (2 graph replays)
#   2. ncu --set full of each hot kernel (one launch, inside the real step),
#      reduced on the box to details / raw CSVs + a stall summary (the
#      .ncu-rep files are deleted so the results fit gpurun's copy-back)
# Usage: bash tools/profile_round.sh <tag> [kernel regex ...]
set -u
TAG=${1:-r1}
shift || true
OUT=gpurun_out/prof_${TAG}
mkdir -p "$OUT"
LS2_PROFILE_RANGE=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --profile-from-start off --csv --log-file "$OUT/bench_launches.csv" \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > "$OUT/bench_under_ncu.log" 2>&1
python tools/launch_summary.py "$OUT/bench_launches.csv" > "$OUT/bench_launches_summary.txt" 2>&1
for K in "$@"; do
  N=$(echo "$K" | tr -c 'A-Za-z0-9_' '_')
  ncu --set full --import-source on --clock-control none --profile-from-start off \
    -k "regex:$K" -c 1 -o "$OUT/$N" python tools/profile_step.py > /dev/null 2>&1
  if [ -f "$OUT/$N.ncu-rep" ]; then
    ncu -i "$OUT/$N.ncu-rep" --page details --csv > "$OUT/ncu_full_$N.csv" 2>/dev/null
    python tools/ncu_details.py "$OUT/ncu_full_$N.csv" > "$OUT/ncu_full_$N.txt" 2>&1
    python tools/ncu_stalls.py "$OUT/$N.ncu-rep" >> "$OUT/ncu_full_$N.txt" 2>&1
    rm -f "$OUT/$N.ncu-rep"
  fi
done
