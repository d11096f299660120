#!/usr/bin/env bash
# GPU pass: parity tests (incl. full-size), then the default bench (S3DIS) and
# the reference arm.  Usage: gpurun -- 'bash tools/gpu_round2a.sh'
set -u
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/r2a_smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/r2a_pytest.txt 2>&1
echo "pytest exit $?" >> $OUT/r2a_pytest.txt
timeout 900 python bench.py --steps 5 --warmup 3 > $OUT/r2a_bench.json 2> $OUT/r2a_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/r2a_ref.json 2> $OUT/r2a_ref.err
tail -3 $OUT/r2a_pytest.txt
cat $OUT/r2a_bench.json $OUT/r2a_ref.json
