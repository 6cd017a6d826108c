#!/bin/bash
# A/B: pass-0 segment length from the position table; parity of the variant
set -u
for cfg in C3 C4 C2 C5; do
  echo "== $cfg"; bash tools/variant_run.sh $cfg lp0 lp1 lp0 lp1
done
PBIT_LIB_PATH=build/var/libpbit_lp1.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -m gpu -x -q 2>&1 | tail -2
