#!/bin/bash
# round 2 (re-entry): relink partition with the next tile's bin claims issued before the
# current tile's write-out (PBIT_PART_PIPE); parity of the bounds-checked variant first
set -u
mkdir -p gpurun_out/r2ao
python tests/fake_nccl/build_fake.py > /dev/null
PBIT_BOUNDS_CHECK=1 PBIT_LIB_PATH=build/var/libpbit_partpipe_bounds.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -m gpu -x -q > gpurun_out/r2ao/parity_bounds.log 2>&1; echo parity rc=$?; tail -1 gpurun_out/r2ao/parity_bounds.log
PBIT_LIB_PATH=build/var/libpbit_partpipe.so timeout 200 python tools/fuzz_parity.py 90 5151 > gpurun_out/r2ao/fuzz.log 2>&1; echo fuzz rc=$?; tail -1 gpurun_out/r2ao/fuzz.log
for cfg in C3 C2 C4 C5; do
  echo "== $cfg"; bash tools/variant_run.sh $cfg main partpipe main partpipe
done 2>&1 | tee gpurun_out/r2ao/variants.log
# the multi-GPU harness links its own library: flip the default in this scratch copy
sed -i 's/^#define PBIT_PART_PIPE 0$/#define PBIT_PART_PIPE 1/' paper_cs_0511020_b200/csrc/kernels.cuh
python tests/fake_nccl/build_fake.py -f > /dev/null && python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_mg_threads.py tests/test_gpu_mg.py -m gpu -x -q > gpurun_out/r2ao/mg.log 2>&1; echo mg rc=$?; tail -1 gpurun_out/r2ao/mg.log
PBIT_MG_TRANSPORT=peer timeout 150 python tests/fake_nccl/fuzz_mg.py 60 777 > gpurun_out/r2ao/fuzz_mg_peer.log 2>&1; echo fuzz_mg rc=$?; tail -1 gpurun_out/r2ao/fuzz_mg_peer.log
