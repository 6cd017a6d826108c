#!/bin/bash
set -u
mkdir -p gpurun_out/r2e
python tests/fake_nccl/build_fake.py > /dev/null
timeout 900 python -m pytest tests/test_gpu_mg.py tests/test_gpu_mg_threads.py -q > gpurun_out/r2e/mg.log 2>&1; echo mg rc=$?; tail -3 gpurun_out/r2e/mg.log
grep -h "ok (\|FAILED\|differs" gpurun_out/r2e/mg.log | head
python tools/mg_one_rank.py C3
PBIT_MG_TRANSPORT=nccl python tools/mg_one_rank.py C3
python tools/mg_one_rank.py C2
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/r2e/parity.log 2>&1; echo parity rc=$?; tail -2 gpurun_out/r2e/parity.log
timeout 600 python bench.py > gpurun_out/r2e/bench.json 2> gpurun_out/r2e/bench.err; echo bench rc=$?
python -c "import json; d=json.load(open('gpurun_out/r2e/bench.json')); print(d['ms_per_step'], d['roofline']['phase_ms'], d['cpu_baseline'], d['e2e'])"
