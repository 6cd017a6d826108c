#!/bin/bash
# longer fuzz runs of the release build: single GPU, and the multi-rank harness with every transport
set -u
mkdir -p gpurun_out/r2p
python tests/fake_nccl/build_fake.py > /dev/null
timeout 720 python tools/fuzz_parity.py 600 4242 > gpurun_out/r2p/fuzz.log 2>&1; echo fuzz rc=$?; tail -1 gpurun_out/r2p/fuzz.log
for t in hybrid peer nccl; do PBIT_MG_TRANSPORT=$t timeout 400 python tests/fake_nccl/fuzz_mg.py 300 $RANDOM > gpurun_out/r2p/fuzz_mg_$t.log 2>&1; echo fuzz_mg_$t rc=$?; tail -1 gpurun_out/r2p/fuzz_mg_$t.log; done
