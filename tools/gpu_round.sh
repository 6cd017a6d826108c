#!/bin/bash
# Round-end evidence on one GPU box: smoke, the GPU tests, the default bench line (with
# the CPU oracle baseline), one bench line per config, and the ncu capture of C3.
#   tools/gpu_round.sh <tag>
set -u
tag=${1:-r01}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo bench rc=$?
cat gpurun_out/bench_$tag.json
bash tools/bench_all.sh
timeout 1200 bash tools/profile_round.sh $tag C3 > gpurun_out/prof_$tag.log 2>&1; echo prof rc=$?
tail -3 gpurun_out/prof_$tag.log
