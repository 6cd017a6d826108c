#!/bin/bash
# round-2 final evidence: smoke, GPU suite (release + bounds-checked), fuzzers, bench lines
# of every config, the default bench, ncu launch lists of C2..C5 and the C3 full capture
set -u
mkdir -p gpurun_out/r2af
python tests/fake_nccl/build_fake.py > /dev/null
PBIT_BOUNDS_CHECK=1 python tests/fake_nccl/build_fake.py > /dev/null
[ -f build/var/libpbit_bounds.so ] || python tools/build_variants.py bounds=-DPBIT_BOUNDS_CHECK=1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2af/smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/r2af/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2af/gpu_all.log 2>&1; echo gpu_all rc=$?; tail -1 gpurun_out/r2af/gpu_all.log
PBIT_BOUNDS_CHECK=1 PBIT_LIB_PATH=build/var/libpbit_bounds.so timeout 2000 python -m pytest tests -m gpu -q > gpurun_out/r2af/gpu_all_bounds.log 2>&1; echo gpu_all_bounds rc=$?; tail -1 gpurun_out/r2af/gpu_all_bounds.log
timeout 400 python tools/fuzz_parity.py 300 7171 > gpurun_out/r2af/fuzz.log 2>&1; echo fuzz rc=$?; tail -1 gpurun_out/r2af/fuzz.log
for t in peer nccl hybrid; do PBIT_MG_TRANSPORT=$t timeout 200 python tests/fake_nccl/fuzz_mg.py 120 $RANDOM > gpurun_out/r2af/fuzz_mg_$t.log 2>&1; echo fuzz_mg_$t rc=$?; tail -1 gpurun_out/r2af/fuzz_mg_$t.log; done
bash tools/bench_all.sh > gpurun_out/r2af/bench_all.log 2>&1; cat gpurun_out/r2af/bench_all.log; mv gpurun_out/bench_*.json gpurun_out/r2af/ 2>/dev/null
timeout 600 python bench.py > gpurun_out/r2af/bench.json 2> gpurun_out/r2af/bench.err; echo bench rc=$?
timeout 600 python bench.py --impl reference > gpurun_out/r2af/bench_ref.json 2> gpurun_out/r2af/bench_ref.err; echo bench_ref rc=$?
bash tools/profile_round.sh r2af_C3 C3 > gpurun_out/r2af/prof_C3.log 2>&1; echo prof C3 rc=$?
for cfg in C2 C4 C5; do
  mkdir -p gpurun_out/r2af_$cfg
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      --csv --log-file gpurun_out/r2af_$cfg/launches.csv python tools/prof_run.py --config $cfg > gpurun_out/r2af_$cfg/ncu.log 2>&1
  echo prof $cfg rc=$?
done
