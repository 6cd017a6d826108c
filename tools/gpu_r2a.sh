#!/bin/bash
# round 2, first GPU check: smoke, GPU tests (goldens present so far), bench default and with
# the workspace released after every call
set -u
mkdir -p gpurun_out/r2a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a/smoke.log 2>&1; echo smoke rc=$?
timeout 1800 python -m pytest tests -m gpu -x -q -k "not (golden and (C3 or C4 or C5))" > gpurun_out/r2a/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/r2a/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2a/bench.json 2> gpurun_out/r2a/bench.err; echo bench rc=$?
PBIT_POOL_KEEP_GB=0 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2a/bench_keep0.json 2>> gpurun_out/r2a/bench.err; echo bench0 rc=$?
cut -c1-400 gpurun_out/r2a/bench.json gpurun_out/r2a/bench_keep0.json
