set -u
mkdir -p gpurun_out/v1
python tests/fake_nccl/build_fake.py > /dev/null
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v1/smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/v1/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/v1/gpu_all.log 2>&1; echo gpu_all rc=$?; tail -2 gpurun_out/v1/gpu_all.log
timeout 600 python bench.py > gpurun_out/v1/bench.json 2> gpurun_out/v1/bench.err; echo bench rc=$?
cat gpurun_out/v1/bench.json
