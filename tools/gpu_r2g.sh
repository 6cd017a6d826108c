#!/bin/bash
set -u
mkdir -p gpurun_out/r2g
python tests/fake_nccl/build_fake.py > /dev/null
timeout 3000 python -m pytest tests -m gpu -q > gpurun_out/r2g/gpu_all.log 2>&1; echo gpu_all rc=$?; tail -5 gpurun_out/r2g/gpu_all.log
grep -h "FAILED" gpurun_out/r2g/gpu_all.log | head
for t in peer nccl; do PBIT_MG_TRANSPORT=$t timeout 900 python tests/fake_nccl/run_mg_threads.py > gpurun_out/r2g/mg_$t.log 2>&1; echo mg_$t rc=$?; tail -6 gpurun_out/r2g/mg_$t.log; done
