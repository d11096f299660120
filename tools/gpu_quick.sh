#!/usr/bin/env bash
# Quick GPU check: the GPU test suite, then S3DIS op timing and short bench
# lines for the given configs.  bash tools/gpu_quick.sh [config ...]
set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/quick_pytest.txt 2>&1
echo "pytest exit $?"; tail -3 $OUT/quick_pytest.txt
PCP_OP_TIMING=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-kernel-pass 2>/dev/null | tail -1 | \
  python -c "import json,sys; d=json.loads(sys.stdin.read()); print('optiming', round(d['value']), d.get('op_cycle_share'), d.get('voxel_phase_share'))"
for c in "$@"; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-kernel-pass 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['value']), 'e2e', d['e2e'] and round(d['e2e']['value']), d['clocks'])"
done
