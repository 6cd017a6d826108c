#!/bin/bash
# One bench line per BASELINE config and the paper-shaped context workload (K = 4, the
# paper's, and K = 8); context for DESIGN.md -- the driver's line is C3.
mkdir -p gpurun_out
for spec in C1 C2 C3 C4 C5 ctx ctx:8; do
  cfg=${spec%%:*}; kk=""; [[ "$spec" == *:* ]] && kk="--digit-bits ${spec#*:}"
  f=gpurun_out/bench_${spec/:/_K}
  timeout 900 python bench.py --config $cfg $kk --steps 5 --warmup 3 --no-cpu-baseline > $f.json 2> $f.err
  echo "$spec rc=$? $(python -c "import json; d=json.load(open('$f.json')); print(round(d['ms_per_step'],3), 'ms', round(d['value']/1e9,3), 'G nodes/s', {k: round(v,3) for k,v in d['roofline']['phase_ms'].items()})" 2>&1 | tail -1)"
done
