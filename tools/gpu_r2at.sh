#!/bin/bash
# round 2 (re-entry 5): the pipelined relink partition WITH the proxy fence before the refill
# (PBIT_PART_PIPE=1, PBIT_PP_DBG=1): the failing case 10 times, parity + goldens on its
# bounds-checked build, fuzz with sizes above the one-tile-per-CTA range, and its phase times
set -u
mkdir -p gpurun_out/r2at
T='tests/test_gpu_parity.py::test_ragged_shapes_vs_oracle'
for i in 1 2 3 4 5 6 7 8 9 10; do
  r=$(PBIT_LIB_PATH=build/var/libpbit_pp1.so timeout 200 python -m pytest "$T" -m gpu -q -k "4194323" 2>&1 | grep -E "entries differ|passed|failed" | tail -2 | tr '\n' ' ')
  echo "pp1 run $i: $r"
done 2>&1 | tee gpurun_out/r2at/repeat_pp1.log
PBIT_BOUNDS_CHECK=1 PBIT_LIB_PATH=build/var/libpbit_pp1_bounds.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -m gpu -q > gpurun_out/r2at/pp1_parity_bounds.log 2>&1; echo pp1_parity rc=$?; tail -1 gpurun_out/r2at/pp1_parity_bounds.log
PBIT_LIB_PATH=build/var/libpbit_pp1.so timeout 120 python tools/fuzz_parity.py 60 7373 > gpurun_out/r2at/pp1_fuzz.log 2>&1; echo pp1_fuzz rc=$?; tail -1 gpurun_out/r2at/pp1_fuzz.log
for cfg in C3 C5; do
  echo "== $cfg"; bash tools/variant_run.sh $cfg main pp1 main pp1
done 2>&1 | tee gpurun_out/r2at/variants.log
