#!/bin/bash
# round 2 (re-entry): pass-kernel variants -- per-digit scan prefixes in registers
# (PBIT_SCAN_REG), lane-parallel TMA gather of even-aligned segments in pass 0
# (PBIT_GATHER_LANEBULK), both; parity of the bounds-checked combined variant first
set -u
mkdir -p gpurun_out/r2am
python tests/fake_nccl/build_fake.py > /dev/null
PBIT_BOUNDS_CHECK=1 PBIT_LIB_PATH=build/var/libpbit_lanebulk_bounds.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -m gpu -x -q > gpurun_out/r2am/parity_both_bounds.log 2>&1; echo parity rc=$?; tail -1 gpurun_out/r2am/parity_both_bounds.log
PBIT_LIB_PATH=build/var/libpbit_both.so timeout 200 python tools/fuzz_parity.py 90 4242 > gpurun_out/r2am/fuzz_both.log 2>&1; echo fuzz rc=$?; tail -1 gpurun_out/r2am/fuzz_both.log
for cfg in C3 C2 C4 C5; do
  echo "== $cfg"; bash tools/variant_run.sh $cfg main both scanreg lanebulk main both
done 2>&1 | tee gpurun_out/r2am/variants.log
