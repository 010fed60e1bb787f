#!/bin/bash
# ncu --set full capture of selected kernels (demangled-name regexes) in one bench step.
# usage: profile_kernel.sh <out-name> <regex> [<regex> ...]   (run only after the bench exited 0)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m paper_2312_17482_b200.build > /dev/null
CMD="python bench.py --config ${CONFIG:-C2} --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_k.log 2>&1 || { echo "plain run failed"; tail gpurun_out/plain_k.log; exit 1; }
name=$1; shift
i=0
for rx in "$@"; do
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$rx" -s 0 -c 1 \
      -o gpurun_out/${name}_$i $CMD > gpurun_out/ncu_${name}_$i.log 2>&1
  echo "ncu $rx rc=$?"
  i=$((i+1))
done
