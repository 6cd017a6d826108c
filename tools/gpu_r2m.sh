#!/bin/bash
set -u
mkdir -p gpurun_out/r2m
python tests/fake_nccl/build_fake.py > /dev/null
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2m/smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/r2m/smoke.log
timeout 3000 python -m pytest tests -m gpu -q > gpurun_out/r2m/gpu_all.log 2>&1; echo gpu_all rc=$?; tail -3 gpurun_out/r2m/gpu_all.log
grep -h "FAILED" gpurun_out/r2m/gpu_all.log | head
timeout 600 python bench.py > gpurun_out/r2m/bench.json 2> gpurun_out/r2m/bench.err; echo bench rc=$?
python -c "import json; d=json.load(open('gpurun_out/r2m/bench.json')); print(d['ms_per_step'], d['value'], d['e2e']['value'], d['cpu_baseline']['value'], d['cpu_baseline'].get('subtree_parallel'), d['roofline']['frac'], d['roofline']['frac_at_method_bytes'])"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2m/bench_ref.json 2>&1; echo ref rc=$?; tail -c 300 gpurun_out/r2m/bench_ref.json
