#!/bin/bash
# pipelined e2e: host threads 2/3/4 on C3
set -u
mkdir -p gpurun_out/r2t
for t in 2 3 4; do
  timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --e2e-threads $t > gpurun_out/r2t/b$t.json 2> gpurun_out/r2t/b$t.err
  echo t=$t rc=$?
  python -c "import json; d=json.load(open('gpurun_out/r2t/b$t.json')); e=d['e2e']; print(d['ms_per_step'], e['value']/1e9, e['pipelined'])"
done
