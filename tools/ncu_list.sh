#!/usr/bin/env bash
# Launch list (per-kernel durations) of a short bench run: bash tools/ncu_list.sh <tag> [bench args...]
set -u
TAG=$1; shift
OUT=gpurun_out
mkdir -p $OUT
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $OUT/${TAG}_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-kernel-pass "$@" > $OUT/${TAG}_ncu_stdout.txt 2>&1
python tools/launch_summary.py $OUT/${TAG}_launches.csv > $OUT/${TAG}_hot.txt 2>&1
cat $OUT/${TAG}_hot.txt | head -60
