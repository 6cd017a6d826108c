#!/bin/bash
# the GPU suite and the fuzzers against the bounds-checked build (compute-sanitizer is closed)
set -u
mkdir -p gpurun_out/r2i
export PBIT_BOUNDS_CHECK=1 PBIT_LIB_PATH=build/var/libpbit_bounds.so
python tests/fake_nccl/build_fake.py > /dev/null
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2i/gpu_all_bounds.log 2>&1; echo gpu_all_bounds rc=$?; tail -3 gpurun_out/r2i/gpu_all_bounds.log
grep -h "FAILED\|bounds check failed" gpurun_out/r2i/gpu_all_bounds.log | head
timeout 420 python tools/fuzz_parity.py 360 777 > gpurun_out/r2i/fuzz_bounds.log 2>&1; echo fuzz rc=$?; tail -2 gpurun_out/r2i/fuzz_bounds.log
PBIT_MG_TRANSPORT=peer timeout 420 python tests/fake_nccl/fuzz_mg.py 300 21 > gpurun_out/r2i/fuzz_mg_peer_bounds.log 2>&1; echo fuzz_mg_peer rc=$?; tail -2 gpurun_out/r2i/fuzz_mg_peer_bounds.log
PBIT_MG_TRANSPORT=nccl timeout 300 python tests/fake_nccl/fuzz_mg.py 200 22 > gpurun_out/r2i/fuzz_mg_nccl_bounds.log 2>&1; echo fuzz_mg_nccl rc=$?; tail -2 gpurun_out/r2i/fuzz_mg_nccl_bounds.log
