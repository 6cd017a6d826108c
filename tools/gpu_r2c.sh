#!/bin/bash
# round 2: peer transport harness, parity with 128-bit stores, goldens, A/B of the stores
set -u
mkdir -p gpurun_out/r2c
python tests/fake_nccl/build_fake.py > /dev/null
PBIT_MG_TRANSPORT=peer timeout 900 python tests/fake_nccl/run_mg_threads.py > gpurun_out/r2c/mg_peer.log 2>&1; echo mg_peer rc=$?
tail -14 gpurun_out/r2c/mg_peer.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2c/smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/r2c/smoke.log
timeout 1800 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/r2c/parity.log 2>&1; echo parity rc=$?; tail -3 gpurun_out/r2c/parity.log
timeout 1800 python -m pytest tests/test_gpu_golden.py -q -k "not C5 and not complete" > gpurun_out/r2c/golden.log 2>&1; echo golden rc=$?; tail -3 gpurun_out/r2c/golden.log
for cfg in C3 C2 C4; do bash tools/variant_run.sh $cfg main novec main novec; done
