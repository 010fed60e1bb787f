#!/bin/bash
# long-attention backward A/B: MB_ATTN_LONG_BWD=v1 vs the default, at C4 / F4 shapes
cd "$(dirname "$0")/.."
for shape in "128 512" "64 1024" "32 2048" "128 512 lognormal"; do
  for v in v1 v2; do
    echo -n "$v "; MB_ATTN_LONG_BWD=$v timeout 120 python scripts/attn_bench.py $shape
  done
done
