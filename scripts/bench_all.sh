#!/bin/bash
# bench lines for C2 (default), C3, C4, C5 on one box; JSON lines into gpurun_out/bench_<cfg>.json
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m paper_2312_17482_b200.build > /dev/null
for c in ${CONFIGS:-C2 C4 C5 C3}; do
  extra=""; [ "$c" != "C2" ] && extra="--no-e2e"
  timeout 900 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 $extra > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  python -c "import json;d=json.load(open('gpurun_out/bench_$c.json'));print('$c', round(d['ms_per_step'],2), 'ms', round(d['value']/1e6,4), 'Mtok/s mfu', round(d['mfu']['datasheet_2.25PF'],4), 'clk', d['clocks']['sm_mhz'], 'roof', round(d['roofline']['frac'] or 0,3))" || tail -3 gpurun_out/bench_$c.err
done
