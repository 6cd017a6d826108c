#!/bin/bash
# round 2 (re-entry): validate HEAD after the ranking / staging changes -- smoke, GPU suite,
# fuzz, default bench + reference arm, C3 launch list and full capture
set -u
mkdir -p gpurun_out/r2al
python tests/fake_nccl/build_fake.py > /dev/null
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2al/smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/r2al/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2al/gpu_all.log 2>&1; echo gpu_all rc=$?; tail -1 gpurun_out/r2al/gpu_all.log
timeout 200 python tools/fuzz_parity.py 150 9191 > gpurun_out/r2al/fuzz.log 2>&1; echo fuzz rc=$?; tail -1 gpurun_out/r2al/fuzz.log
timeout 600 python bench.py > gpurun_out/r2al/bench.json 2> gpurun_out/r2al/bench.err; echo bench rc=$?; cut -c1-600 gpurun_out/r2al/bench.json
timeout 600 python bench.py --impl reference > gpurun_out/r2al/bench_ref.json 2> gpurun_out/r2al/bench_ref.err; echo bench_ref rc=$?
bash tools/profile_round.sh r2al_C3 C3 > gpurun_out/r2al/prof_C3.log 2>&1; echo prof C3 rc=$?
