#!/bin/bash
# round 2 (re-entry) final validation: bounds-checked GPU suite and fuzzers, multi-rank
# fuzz per transport, bench lines of every config, launch lists of C2 / C4 / C5, smoke,
# default bench + reference arm
set -u
mkdir -p gpurun_out/r2an
python tests/fake_nccl/build_fake.py > /dev/null
PBIT_BOUNDS_CHECK=1 python tests/fake_nccl/build_fake.py > /dev/null
python tools/build_variants.py bounds=-DPBIT_BOUNDS_CHECK=1 > /dev/null
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2an/smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/r2an/smoke.log
PBIT_BOUNDS_CHECK=1 PBIT_LIB_PATH=build/var/libpbit_bounds.so timeout 2000 python -m pytest tests -m gpu -q > gpurun_out/r2an/gpu_all_bounds.log 2>&1; echo gpu_all_bounds rc=$?; tail -1 gpurun_out/r2an/gpu_all_bounds.log
for t in peer nccl hybrid; do PBIT_MG_TRANSPORT=$t timeout 150 python tests/fake_nccl/fuzz_mg.py 90 $RANDOM > gpurun_out/r2an/fuzz_mg_$t.log 2>&1; echo fuzz_mg_$t rc=$?; tail -1 gpurun_out/r2an/fuzz_mg_$t.log; done
bash tools/bench_all.sh > gpurun_out/r2an/bench_all.log 2>&1; cat gpurun_out/r2an/bench_all.log; mkdir -p gpurun_out/r2an/bench_all; mv gpurun_out/bench_*.json gpurun_out/r2an/bench_all/ 2>/dev/null
timeout 600 python bench.py > gpurun_out/r2an/bench.json 2> gpurun_out/r2an/bench.err; echo bench rc=$?; cut -c1-300 gpurun_out/r2an/bench.json
for cfg in C2 C4 C5; do
  mkdir -p gpurun_out/r2an_$cfg
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      --csv --log-file gpurun_out/r2an_$cfg/launches.csv python tools/prof_run.py --config $cfg > gpurun_out/r2an_$cfg/ncu.log 2>&1
  echo prof $cfg rc=$?
done
timeout 600 python bench.py --impl reference > gpurun_out/r2an/bench_ref.json 2> gpurun_out/r2an/bench_ref.err; echo bench_ref rc=$?
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r2an/gpu_all.log 2>&1; echo gpu_all rc=$?; tail -1 gpurun_out/r2an/gpu_all.log
bash tools/profile_round.sh r2an_C3 C3 > gpurun_out/r2an/prof_C3.log 2>&1; echo prof C3 rc=$?
