OUT=gpurun_out/sweep; mkdir -p $OUT
run() { tag=$1; shift; env "$@" python bench.py --no-cpu-baseline --no-e2e > $OUT/$tag.json 2> $OUT/$tag.err; echo "$tag $(python -c "import json;print(round(json.load(open('$OUT/$tag.json'))['value']))" 2>/dev/null)" >> $OUT/summary.txt; }
run base X=1
for m in 64 96; do run mt$m PCP_MATCH_THREADS=$m; done
for s in 3 5 6 8; do run slots$s PCP_SLOTS=$s; done
for w in 296 888 1184; do run wb$w PCP_WAVE_BATCHES=$w; done
run wb888s3 PCP_WAVE_BATCHES=888 PCP_SLOTS=3
run wb296s8 PCP_WAVE_BATCHES=296 PCP_SLOTS=8
run base2 X=1
cat $OUT/summary.txt
