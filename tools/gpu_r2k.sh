#!/bin/bash
set -u
mkdir -p gpurun_out/r2k
python tests/fake_nccl/build_fake.py > /dev/null
timeout 2400 python -m pytest tests/test_gpu_mg.py tests/test_gpu_mg_threads.py tests/test_gpu_golden.py -q > gpurun_out/r2k/mg_golden.log 2>&1; echo mg_golden rc=$?; tail -3 gpurun_out/r2k/mg_golden.log
grep -h "FAILED" gpurun_out/r2k/mg_golden.log | head
bash tools/bench_all.sh
