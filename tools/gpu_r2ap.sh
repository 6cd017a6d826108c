#!/bin/bash
# round 2 (re-entry 5): validate HEAD (scan-reg + lane-parallel gather defaults) -- smoke, GPU suite,
# fuzz, default bench + reference arm, C3 launch list and full capture; then measure the
# relink partition with pipelined bin claims (PBIT_PART_PIPE variant), parity first
set -u
mkdir -p gpurun_out/r2ap
python tests/fake_nccl/build_fake.py > /dev/null
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2ap/smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/r2ap/smoke.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r2ap/gpu_all.log 2>&1; echo gpu_all rc=$?; tail -1 gpurun_out/r2ap/gpu_all.log
timeout 150 python tools/fuzz_parity.py 90 4242 > gpurun_out/r2ap/fuzz.log 2>&1; echo fuzz rc=$?; tail -1 gpurun_out/r2ap/fuzz.log
timeout 600 python bench.py > gpurun_out/r2ap/bench.json 2> gpurun_out/r2ap/bench.err; echo bench rc=$?; cut -c1-600 gpurun_out/r2ap/bench.json
timeout 600 python bench.py --impl reference > gpurun_out/r2ap/bench_ref.json 2> gpurun_out/r2ap/bench_ref.err; echo bench_ref rc=$?
# PBIT_PART_PIPE: parity of the bounds-checked variant, fuzz, then phase times
PBIT_BOUNDS_CHECK=1 PBIT_LIB_PATH=build/var/libpbit_partpipe_bounds.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -m gpu -x -q > gpurun_out/r2ap/pp_parity_bounds.log 2>&1; echo pp_parity rc=$?; tail -1 gpurun_out/r2ap/pp_parity_bounds.log
PBIT_LIB_PATH=build/var/libpbit_partpipe.so timeout 120 python tools/fuzz_parity.py 60 5151 > gpurun_out/r2ap/pp_fuzz.log 2>&1; echo pp_fuzz rc=$?; tail -1 gpurun_out/r2ap/pp_fuzz.log
for cfg in C3 C2 C4 C5; do
  echo "== $cfg"; bash tools/variant_run.sh $cfg main partpipe main partpipe
done 2>&1 | tee gpurun_out/r2ap/variants.log
bash tools/profile_round.sh r2ap_C3 C3 > gpurun_out/r2ap/prof_C3.log 2>&1; echo prof C3 rc=$?
