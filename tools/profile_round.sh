#!/bin/bash
# Capture the ncu evidence for one config on the GPU box (run under gpurun):
#   1. the launch list of one pbit_sort_list call (device time + DRAM bytes per launch)
#   2. one `--set full` capture of each distinct hot kernel (raw metrics as CSV)
# Usage: tools/profile_round.sh <tag> <config> [digit_bits]
set -u
tag=$1; cfg=$2; K=${3:-0}
out=gpurun_out/$tag
mkdir -p $out
cmd="python tools/prof_run.py --config $cfg --digit-bits $K"
$cmd > $out/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file $out/launches.csv $cmd > $out/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"k_pack|k_walk|k_gather|k_onesweep|k_relink_part|k_relink_apply|k_rank_walk" -c 14 \
    -o $out/full $cmd > $out/ncu_full.log 2>&1
ncu -i $out/full.ncu-rep --page raw --csv > $out/full_raw.csv 2>/dev/null
ncu -i $out/full.ncu-rep --page details > $out/full_details.txt 2>/dev/null
for k in k_walk k_onesweep; do
  ncu -i $out/full.ncu-rep --page source --csv --print-source sass --kernel-name regex:$k --launch-count 1 \
      > $out/sass_$k.csv 2>/dev/null
done
ls -la $out
du -sh $out
# keep the returned tree under the 64 MiB limit
if [ $(du -sm $out/full.ncu-rep | cut -f1) -gt 40 ]; then rm -f $out/full.ncu-rep; echo "dropped full.ncu-rep (size)"; fi
