#!/usr/bin/env bash
# LZ4 phase 4: page-wide pointer jumping (auto) vs a warp per page (PCP_LZ4_PJ=0)
for c in "$@"; do
  echo "pj   $(PCP_LZ4_PJ=1 BENCH_ARGS=--quantized bash tools/bench_lines.sh $c | cut -c1-60)"
  echo "warp $(PCP_LZ4_PJ=0 BENCH_ARGS=--quantized bash tools/bench_lines.sh $c | cut -c1-60)"
done
