#!/usr/bin/env bash
# One --set full capture of a kernel (regex) from a short bench run, summarised
# to text: bash tools/ncu_full.sh <tag> <kernel-regex> <launch-skip> [bench args...]
set -u
TAG=$1; K=$2; SKIP=$3; shift 3
OUT=gpurun_out
mkdir -p $OUT
timeout 1200 ncu --set full --import-source on --clock-control none -k "regex:$K" -s $SKIP -c 1 \
  -o $OUT/${TAG}_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-kernel-pass "$@" \
  > $OUT/${TAG}_full_stdout.txt 2>&1
ncu -i $OUT/${TAG}_full.ncu-rep --page details --csv > $OUT/${TAG}_details.csv 2>/dev/null
ncu -i $OUT/${TAG}_full.ncu-rep --page source --csv --print-source sass > $OUT/${TAG}_source.csv 2>/dev/null
ncu -i $OUT/${TAG}_full.ncu-rep --page source --csv --print-source cuda > $OUT/${TAG}_cuda.csv 2>/dev/null
python tools/ncu_hot.py $OUT/${TAG}_source.csv 25 > $OUT/${TAG}_hot.txt 2>&1
grep -E "Duration|DRAM Throughput|Memory Throughput|Achieved Occupancy|Registers Per|Warp Cycles Per Issued|Issue Slots Busy|L2 Hit Rate|L1/TEX Hit" $OUT/${TAG}_details.csv | head -30
head -40 $OUT/${TAG}_hot.txt
rm -f $OUT/${TAG}_full.ncu-rep
