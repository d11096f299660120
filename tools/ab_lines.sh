#!/usr/bin/env bash
# A/B bench lines: current tree vs ab/base (a worktree of the previous build),
# interleaved, for the given configs.  bash tools/ab_lines.sh s3dis shapenet_part ...
for c in "$@"; do
  echo "new  $(bash tools/bench_lines.sh $c | cut -c1-60)"
  echo "base $(cd ab/base && bash ../../tools/bench_lines.sh $c | cut -c1-60)"
done
