#!/bin/bash
set -u
mkdir -p gpurun_out/r2f
python tests/fake_nccl/build_fake.py > /dev/null
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r2f/gpu_all.log 2>&1; echo gpu_all rc=$?; tail -5 gpurun_out/r2f/gpu_all.log
grep -h "ok (\|FAILED" gpurun_out/r2f/gpu_all.log | head
python tools/mg_one_rank.py C3
python tools/mg_one_rank.py C5
