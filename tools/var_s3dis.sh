#!/usr/bin/env bash
# S3DIS bench variance under environment variants: bash tools/var_s3dis.sh "A=1" "PCP_SLOTS=3" ...
for v in "$@"; do
  for i in 1 2 3; do
    echo "[$v] $(env $v timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-kernel-pass 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],1))")"
  done
done
