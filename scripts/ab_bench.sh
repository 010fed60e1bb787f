#!/bin/bash
# Alternate bench runs of ab/libmosaicbert_<a>.so and the in-tree build on one box (same clocks and
# thermals for both); prints ms_per_step per run.   usage: ab_bench.sh <a-name> [rounds] [bench args]
cd "$(dirname "$0")/.."
a=$1; rounds=${2:-2}; shift 2
for i in $(seq 1 $rounds); do
  for v in "$a" new; do
    if [ "$v" = new ]; then lib=""; else lib="ab/libmosaicbert_$v.so"; fi
    MB_LIBRARY=$lib python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e "$@" > gpurun_out/ab_$v.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/ab_$v.json'));print('$v', round(d['ms_per_step'],3), d['clocks']['sm_mhz'])"
  done
done
