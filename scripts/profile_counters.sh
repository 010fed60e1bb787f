#!/bin/bash
# Per-launch ncu counters (duration, DRAM bytes, tensor-pipe / SM / DRAM utilisation) for every kernel
# of one bench step; run only after the same command exited 0.   usage: profile_counters.sh <config> <out.csv>
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CMD="python bench.py --config $1 --accum 1 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_cnt.log 2>&1 || { echo "plain run failed"; exit 1; }
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/$2 $CMD > gpurun_out/ncu_cnt.log 2>&1
echo "ncu rc=$?"
