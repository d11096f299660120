#!/usr/bin/env bash
# One GPU box pass that refreshes every committed number: bench lines for all
# five configs + the reference arm, ncu launch lists (gpu__time_duration per
# launch) and one --set full capture of the dominant kernels per config,
# summarised by tools/ncu_summary.py into gpurun_out/ (copy to profiles/).
# Reports are deleted on the box after summarising (gpurun_out <= 64 MiB).
#   gpurun --timeout 3000 -- 'bash tools/measure_round.sh <tag>'
set -u
TAG=${1:-round1}
OUT=gpurun_out
B=$(cat .build_id 2>/dev/null || git rev-parse --short HEAD 2>/dev/null || echo unknown)
mkdir -p $OUT
nproc > $OUT/${TAG}_nproc.txt
python bench.py > $OUT/${TAG}_default.json 2> $OUT/${TAG}_default.err
for c in modelnet40 kitti s3dis scannet; do
  python bench.py --config $c > $OUT/${TAG}_$c.json 2> $OUT/${TAG}_$c.err
done
python bench.py --impl reference > $OUT/${TAG}_ref.json 2> $OUT/${TAG}_ref.err

# C2: launch list over a short run, full set on the decode pair + k_cloud of one wave
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/${TAG}_c2_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none \
  -k 'regex:k_page_decode|k_page_matches|k_cloud' -s 3 -c 3 -o $OUT/${TAG}_c2_full \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python tools/ncu_summary.py $OUT/${TAG}_c2_launches.csv $OUT/${TAG}_c2_full.ncu-rep shapenet_part \
  $OUT/${TAG}_c2_ncu_summary.md "Command: \`python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e\` (launch list) and \`--steps 1 --warmup 1\` with \`-k regex:k_page_decode|k_page_matches|k_cloud -s 3 -c 3\` (full set). B200, build $B. One wave = 18944 clouds." 18944 > /dev/null
rm -f $OUT/${TAG}_c2_full.ncu-rep

for c in modelnet40 kitti s3dis scannet; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/${TAG}_${c}_launches.csv \
    python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_cloud -s 1 -c 2 \
    -o $OUT/${TAG}_${c}_full \
    python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --clouds-per-gpu 148 > /dev/null 2>&1
  python tools/ncu_summary.py $OUT/${TAG}_${c}_launches.csv $OUT/${TAG}_${c}_full.ncu-rep $c \
    $OUT/${TAG}_${c}_ncu_summary.md "Command: \`python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e\` (launch list) and \`--steps 1 --warmup 1 --clouds-per-gpu 148\` with \`-k regex:k_cloud -s 1 -c 2\` (full set, one 148-cloud wave). B200, build $B." 148 > /dev/null
  rm -f $OUT/${TAG}_${c}_full.ncu-rep
done
cp profiles/ncu_summary.json $OUT/${TAG}_ncu_summary.json 2>/dev/null
echo done
