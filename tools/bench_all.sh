#!/bin/bash
# One bench line per BASELINE config (context for DESIGN.md; the driver's line is C3).
mkdir -p gpurun_out
for cfg in C1 C2 C3 C4 C5; do
  timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err
  echo "$cfg rc=$? $(python -c "import json; d=json.load(open('gpurun_out/bench_$cfg.json')); print(round(d['ms_per_step'],3), 'ms', round(d['value']/1e9,3), 'G nodes/s', {k: round(v,3) for k,v in d['roofline']['phase_ms'].items()})" 2>&1 | tail -1)"
done
