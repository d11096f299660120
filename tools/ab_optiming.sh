#!/usr/bin/env bash
# A/B of S3DIS k_cloud op timing under environment variants:
#   bash tools/ab_optiming.sh "" "PCP_NO_RING=1" ...
for v in "$@"; do
  env $v PCP_OP_TIMING=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-kernel-pass ${BENCH_ARGS:-} 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$v]', round(d['value']), d.get('op_cycle_share'), d.get('voxel_phase_share'))"
done
