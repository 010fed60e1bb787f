#!/bin/bash
# run GPU test groups in separate processes, each under its own timeout
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt 2>&1
python -m paper_2312_17482_b200.build > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for k in "$@"; do
  echo "=== $k" >> gpurun_out/tests.log
  timeout 600 python -m pytest tests -m gpu -q -k "$k" -p no:cacheprovider >> gpurun_out/tests.log 2>&1
  echo "exit $?" >> gpurun_out/tests.log
done
tail -c 20000 gpurun_out/tests.log
