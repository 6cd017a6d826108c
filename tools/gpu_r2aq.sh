#!/bin/bash
# round 2 (re-entry 5, final): validate HEAD after a default flip -- smoke, GPU suite (release),
# parity + goldens on the bounds-checked build, fuzz, default bench + reference arm, C3 launch list
set -u
mkdir -p gpurun_out/r2aq
python tests/fake_nccl/build_fake.py > /dev/null
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2aq/smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/r2aq/smoke.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r2aq/gpu_all.log 2>&1; echo gpu_all rc=$?; tail -1 gpurun_out/r2aq/gpu_all.log
timeout 600 python bench.py > gpurun_out/r2aq/bench.json 2> gpurun_out/r2aq/bench.err; echo bench rc=$?; cut -c1-600 gpurun_out/r2aq/bench.json
timeout 600 python bench.py --impl reference > gpurun_out/r2aq/bench_ref.json 2> gpurun_out/r2aq/bench_ref.err; echo bench_ref rc=$?
timeout 150 python tools/fuzz_parity.py 90 6262 > gpurun_out/r2aq/fuzz.log 2>&1; echo fuzz rc=$?; tail -1 gpurun_out/r2aq/fuzz.log
PBIT_BOUNDS_CHECK=1 PBIT_LIB_PATH=build/var/libpbit_bounds.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -m gpu -x -q > gpurun_out/r2aq/parity_bounds.log 2>&1; echo parity_bounds rc=$?; tail -1 gpurun_out/r2aq/parity_bounds.log
bash tools/profile_round.sh r2aq_C3 C3 > gpurun_out/r2aq/prof_C3.log 2>&1; echo prof C3 rc=$?
