#!/bin/bash
set -u
mkdir -p gpurun_out/r2h
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -k "host or invalid or prev or small" > gpurun_out/r2h/parity_host.log 2>&1; echo parity_host rc=$?; tail -3 gpurun_out/r2h/parity_host.log
timeout 600 python bench.py > gpurun_out/r2h/bench.json 2> gpurun_out/r2h/bench.err; echo bench rc=$?
python -c "import json; d=json.load(open('gpurun_out/r2h/bench.json')); print(d['ms_per_step'], d['e2e'], d['roofline']['phase_ms'])"
timeout 600 python bench.py --config C2 --no-cpu-baseline > gpurun_out/r2h/bench_C2.json 2>&1; python -c "import json; d=json.load(open('gpurun_out/r2h/bench_C2.json')); print('C2', d['ms_per_step'], d['e2e'])"
