# Slot-count sweep over every config (diagnostics): PCP_SLOTS=4 vs 5 vs 6, no CPU/e2e legs
OUT=gpurun_out/sweep_slots; mkdir -p $OUT
for c in shapenet_part modelnet40 kitti s3dis scannet; do
  for s in 4 5 6 4b 5b; do
    PCP_SLOTS=${s%b} python bench.py --config $c --no-cpu-baseline --no-e2e > $OUT/${c}_$s.json 2> $OUT/${c}_$s.err
    echo "$c $s $(python -c "import json;print(round(json.load(open('$OUT/${c}_$s.json'))['value']))" 2>/dev/null)" >> $OUT/summary.txt
  done
done
cat $OUT/summary.txt
