#!/usr/bin/env bash
# vx stage check: its tests, the full-size parity tests, then the S3DIS bench.
set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_voxel_wave.py -x -q -p no:cacheprovider > $OUT/vx_pytest.txt 2>&1
echo "exit $?" >> $OUT/vx_pytest.txt
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_pipeline.py -x -q -p no:cacheprovider > $OUT/vx_pytest2.txt 2>&1
echo "exit $?" >> $OUT/vx_pytest2.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $OUT/vx_bench.json 2> $OUT/vx_bench.err
tail -15 $OUT/vx_pytest.txt; tail -3 $OUT/vx_pytest2.txt; cat $OUT/vx_bench.json; tail -5 $OUT/vx_bench.err
