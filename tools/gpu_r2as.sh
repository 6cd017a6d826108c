#!/bin/bash
# round 2 (re-entry 5): bisect the PBIT_PART_PIPE race with the PBIT_PP_DBG knobs
# (1 proxy fence before the refill, 2 claims after the write-out, 4 fully serial), 4 runs each
set -u
mkdir -p gpurun_out/r2as
T='tests/test_gpu_parity.py::test_ragged_shapes_vs_oracle'
for v in "$@"; do
  for i in 1 2 3 4; do
    r=$(PBIT_LIB_PATH=build/var/libpbit_$v.so timeout 200 python -m pytest "$T" -m gpu -q -k "4194323" 2>&1 | grep -E "entries differ|passed|failed" | tail -2 | tr '\n' ' ')
    echo "$v run $i: $r"
  done
done 2>&1 | tee gpurun_out/r2as/bisect_$1.log
