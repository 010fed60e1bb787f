#!/bin/bash
# full GPU suite, one process per test file (each under its own timeout), then the default bench line
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt 2>&1
python -m paper_2312_17482_b200.build > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
: > gpurun_out/tests.log
for f in ${FILES:-tests/test_gpu_kernels.py tests/test_gpu_model.py tests/test_gpu_dp.py tests/test_gpu_fullsize.py tests/test_gpu_determinism.py}; do
  echo "=== $f" >> gpurun_out/tests.log
  timeout ${TT:-900} python -m pytest $f -m gpu -q -rf -p no:cacheprovider ${PYARGS} >> gpurun_out/tests.log 2>&1
  echo "exit $?" >> gpurun_out/tests.log
done
if [ -z "$NOBENCH" ]; then
  timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/tests.log
fi
grep -E "===|passed|failed|exit|FAILED|Error" gpurun_out/tests.log | tail -60
