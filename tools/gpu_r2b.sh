#!/bin/bash
# round 2: multi-rank harness (both transports), 1-rank NCCL, parity, goldens, bench
set -u
mkdir -p gpurun_out/r2b
cd $GRAFT_REPO_ROOT 2>/dev/null || true
python tests/fake_nccl/build_fake.py > /dev/null
PBIT_MG_TRANSPORT=peer timeout 900 python tests/fake_nccl/run_mg_threads.py > gpurun_out/r2b/mg_peer.log 2>&1; echo mg_peer rc=$?
tail -14 gpurun_out/r2b/mg_peer.log
PBIT_MG_TRANSPORT=nccl timeout 900 python tests/fake_nccl/run_mg_threads.py > gpurun_out/r2b/mg_nccl.log 2>&1; echo mg_nccl rc=$?
tail -14 gpurun_out/r2b/mg_nccl.log
timeout 600 python -m pytest tests/test_gpu_mg.py -q > gpurun_out/r2b/gpu_mg.log 2>&1; echo gpu_mg rc=$?; tail -3 gpurun_out/r2b/gpu_mg.log
timeout 1800 python -m pytest tests/test_gpu_parity.py -q > gpurun_out/r2b/parity.log 2>&1; echo parity rc=$?; tail -5 gpurun_out/r2b/parity.log
timeout 1800 python -m pytest tests/test_gpu_golden.py -q -k "not C5" > gpurun_out/r2b/golden.log 2>&1; echo golden rc=$?; tail -5 gpurun_out/r2b/golden.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2b/bench.json 2> gpurun_out/r2b/bench.err; echo bench rc=$?
python -c "import json; d=json.load(open('gpurun_out/r2b/bench.json')); print(d['ms_per_step'], d['roofline']['phase_ms'])"
