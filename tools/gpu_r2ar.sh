#!/bin/bash
# round 2 (re-entry 5): is the PBIT_PART_PIPE parity failure the variant's, and is it deterministic?
# The failing case, 6 times against each of: main release, main bounds, partpipe release, partpipe bounds.
set -u
mkdir -p gpurun_out/r2ar
T='tests/test_gpu_parity.py::test_ragged_shapes_vs_oracle'
for lib in paper_cs_0511020_b200/libpbit.so build/var/libpbit_bounds.so build/var/libpbit_partpipe.so build/var/libpbit_partpipe_bounds.so; do
  for i in 1 2 3 4 5 6; do
    r=$(PBIT_LIB_PATH=$lib timeout 200 python -m pytest "$T" -m gpu -q -k "4194323" 2>&1 | grep -E "entries differ|passed|failed" | tail -2 | tr '\n' ' ')
    echo "$lib run $i: $r"
  done
done 2>&1 | tee gpurun_out/r2ar/repeat.log
