#!/usr/bin/env bash
# Round-2 measurement pass: bench lines for all five configs (raw float and
# quantized / LZ4 pages), the reference arm per config, and ncu evidence
# (launch list + one --set full capture) for the default (S3DIS) and C2.
#   gpurun --timeout 5400 -- 'bash tools/measure_round2.sh r2'
set -u
TAG=${1:-r2}
OUT=gpurun_out/$TAG
mkdir -p $OUT
B=$(cat .build_id 2>/dev/null || echo unknown)  # written by the caller before gpurun (no .git on the box)
nproc > $OUT/nproc.txt
lscpu | grep -E "Model name|^CPU\(s\)" > $OUT/lscpu.txt 2>/dev/null
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt 2>&1
python bench.py > $OUT/s3dis.json 2> $OUT/s3dis.err
python bench.py --impl reference > $OUT/ref_s3dis.json 2> $OUT/ref_s3dis.err
python bench.py --quantized > $OUT/s3dis_q.json 2> $OUT/s3dis_q.err
for c in shapenet_part modelnet40 kitti scannet; do
  python bench.py --config $c > $OUT/$c.json 2> $OUT/$c.err
  python bench.py --config $c --quantized > $OUT/${c}_q.json 2> $OUT/${c}_q.err
  python bench.py --config $c --impl reference --steps 3 --warmup 1 > $OUT/ref_$c.json 2> $OUT/ref_$c.err
done
# ncu: launch lists (short runs) and one full-set capture of the dominant kernel
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $OUT/s3dis_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-kernel-pass > /dev/null 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_cloud -s 1 -c 1 -o $OUT/s3dis_full \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-kernel-pass --clouds-per-gpu 148 > /dev/null 2>&1
python tools/ncu_summary.py $OUT/s3dis_launches.csv $OUT/s3dis_full.ncu-rep s3dis $OUT/s3dis_ncu_summary.md \
  "Commands: \`python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-kernel-pass\` (launch list, 256-room waves) and the same with \`--clouds-per-gpu 148\` under \`ncu --set full -k regex:k_cloud -s 1 -c 1\` (one 148-room wave). B200, build $B." 148 > /dev/null 2>&1
rm -f $OUT/s3dis_full.ncu-rep
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $OUT/c2_launches.csv python bench.py --config shapenet_part --steps 1 --warmup 2 --no-cpu-baseline --no-e2e --no-kernel-pass > /dev/null 2>&1
python tools/launch_summary.py $OUT/s3dis_launches.csv > $OUT/s3dis_launch_summary.txt 2>&1
python tools/launch_summary.py $OUT/c2_launches.csv > $OUT/c2_launch_summary.txt 2>&1
cp profiles/ncu_summary.json $OUT/ncu_summary.json 2>/dev/null
for f in $OUT/*.json; do echo "== $f"; head -c 600 $f; echo; done
