#!/bin/bash
# evidence after the L2-prefetch changes: smoke, GPU suite, fuzz, bench, C3 ncu launch list + full capture
set -u
mkdir -p gpurun_out/r2ab
python tests/fake_nccl/build_fake.py > /dev/null
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2ab/smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/r2ab/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2ab/gpu_all.log 2>&1; echo gpu_all rc=$?; tail -2 gpurun_out/r2ab/gpu_all.log
timeout 300 python tools/fuzz_parity.py 180 9191 > gpurun_out/r2ab/fuzz.log 2>&1; echo fuzz rc=$?; tail -1 gpurun_out/r2ab/fuzz.log
timeout 600 python bench.py > gpurun_out/r2ab/bench.json 2> gpurun_out/r2ab/bench.err; echo bench rc=$?
bash tools/profile_round.sh r2ab_C3 C3 > gpurun_out/r2ab/prof.log 2>&1; echo prof rc=$?
