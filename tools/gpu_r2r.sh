#!/bin/bash
# final validation of the round: smoke, the GPU suite (release and bounds-checked builds), bench
set -u
mkdir -p gpurun_out/r2r
python tests/fake_nccl/build_fake.py > /dev/null
PBIT_BOUNDS_CHECK=1 python tests/fake_nccl/build_fake.py > /dev/null
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2r/smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/r2r/smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2r/gpu_all.log 2>&1; echo gpu_all rc=$?; tail -2 gpurun_out/r2r/gpu_all.log
PBIT_BOUNDS_CHECK=1 PBIT_LIB_PATH=build/var/libpbit_bounds.so timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2r/gpu_all_bounds.log 2>&1; echo gpu_all_bounds rc=$?; tail -2 gpurun_out/r2r/gpu_all_bounds.log
grep -h "FAILED" gpurun_out/r2r/gpu_all*.log | head
timeout 600 python bench.py > gpurun_out/r2r/bench.json 2> gpurun_out/r2r/bench.err; echo bench rc=$?
python -c "import json; d=json.load(open('gpurun_out/r2r/bench.json')); print(d['ms_per_step'], d['value'], d['e2e']['value'], d['roofline']['frac'], d['clocks'])"
