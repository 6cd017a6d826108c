#!/bin/bash
# Phase times of library variants (build/var/libpbit_<name>.so) on one config:
#   tools/variant_run.sh <config> <name[:ENV=V]> ...
cfg=$1; shift
for spec in "$@"; do
  name=${spec%%:*}; envs=""
  [[ "$spec" == *:* ]] && envs=${spec#*:}
  lib=build/var/libpbit_$name.so; [ "$name" = "main" ] && lib=paper_cs_0511020_b200/libpbit.so
  out=$(env $envs PBIT_LIB_PATH=$lib timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --e2e-threads 0 2>&1 | tail -1)
  echo "$spec: $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), {k: round(v,3) for k,v in d["roofline"]["phase_ms"].items()})' 2>/dev/null || echo "$out" | tail -c 300)"
done
