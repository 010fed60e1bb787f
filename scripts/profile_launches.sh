#!/bin/bash
# ncu launch list (device time per kernel) of one bench step; run only after the same command exited 0.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m paper_2312_17482_b200.build > /dev/null
CMD="python bench.py --config ${CONFIG:-C2} --accum 1 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu.log 2>&1
echo "ncu rc=$?"
tail -3 gpurun_out/ncu.log
