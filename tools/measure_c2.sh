#!/usr/bin/env bash
# Headline-only refresh (C2): bench line, ncu launch list and the full-set
# summary of the decode pair + k_cloud, into gpurun_out/ (copy to profiles/).
#   gpurun --timeout 1500 -- 'bash tools/measure_c2.sh <tag>'
set -u
TAG=${1:-round1}
OUT=gpurun_out
B=$(cat .build_id 2>/dev/null || echo unknown)
mkdir -p $OUT
python bench.py > $OUT/${TAG}_default.json 2> $OUT/${TAG}_default.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/${TAG}_c2_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none \
  -k 'regex:k_page_decode|k_page_matches|k_cloud' -s 3 -c 3 -o $OUT/${TAG}_c2_full \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python tools/ncu_summary.py $OUT/${TAG}_c2_launches.csv $OUT/${TAG}_c2_full.ncu-rep shapenet_part \
  $OUT/${TAG}_c2_ncu_summary.md "Command: \`python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e\` (launch list) and \`--steps 1 --warmup 1\` with \`-k regex:k_page_decode|k_page_matches|k_cloud -s 3 -c 3\` (full set). B200, build $B. One wave = 18944 clouds." 18944 > /dev/null
rm -f $OUT/${TAG}_c2_full.ncu-rep
cp profiles/ncu_summary.json $OUT/${TAG}_ncu_summary.json 2>/dev/null
echo done
