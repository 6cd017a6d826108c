#!/bin/bash
# round-2 ncu evidence: C3 launch list + full capture of the hot kernels; launch lists of
# C2 / C4 / C5; the 1-rank multi-GPU call (peer transport) on C3
set -u
timeout 1500 bash tools/profile_round.sh r02 C3 > gpurun_out/prof_r02.log 2>&1; echo prof rc=$?; tail -3 gpurun_out/prof_r02.log
for cfg in C2 C4 C5; do
  out=gpurun_out/r02_$cfg; mkdir -p $out
  python tools/prof_run.py --config $cfg > $out/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      --csv --log-file $out/launches.csv python tools/prof_run.py --config $cfg > $out/ncu.log 2>&1; echo $cfg rc=$?
done
out=gpurun_out/r02_mg1_C3; mkdir -p $out
python tools/mg_prof_run.py C3 > $out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file $out/launches.csv python tools/mg_prof_run.py C3 > $out/ncu.log 2>&1; echo mg1 rc=$?
du -sh gpurun_out/r02*
