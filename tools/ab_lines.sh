#!/usr/bin/env bash
# A/B bench lines: current tree vs ab/base (a worktree of the previous build),
# interleaved, for the given configs.  bash tools/ab_lines.sh s3dis shapenet_part ...
show() { python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], round(d['value']), 'e2e', round(d['e2e']['value']), 'sm_mhz', d['clocks']['sm_mhz'], d['clocks']['reasons'])"; }
for c in "$@"; do
  echo "new  $(timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-kernel-pass 2>/dev/null | tail -1 | show)"
  echo "base $(cd ab/base && timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-kernel-pass 2>/dev/null | tail -1 | show)"
done
