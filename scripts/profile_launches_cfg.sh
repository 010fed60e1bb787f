#!/bin/bash
# ncu launch list (device time per kernel) of one bench step of a given config; run only after the
# same command exited 0.   usage: profile_launches_cfg.sh <config> <out.csv>
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m paper_2312_17482_b200.build > /dev/null
CMD="python bench.py --config $1 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_$1.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$2 $CMD > gpurun_out/ncu_$1.log 2>&1
echo "ncu rc=$?"
