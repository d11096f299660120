#!/usr/bin/env bash
# Short bench lines (value, e2e, PCIe fraction) for the given configs:
#   bash tools/bench_lines.sh shapenet_part s3dis ...   (BENCH_ARGS adds flags)
for c in "$@"; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-kernel-pass ${BENCH_ARGS:-} 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('$c', round(d['value']), 'e2e', e and round(e['value']), e and e.get('pcie'))"
done
