#!/bin/bash
# Full ncu capture of ONE launch of a kernel in one C3 call + its SASS source page:
#   tools/ncu_one.sh <kernel regex> <launch-skip> <tag> [config]
set -u
re=$1; skip=$2; tag=$3; cfg=${4:-C3}
mkdir -p gpurun_out/$tag
python tools/prof_run.py --config $cfg > gpurun_out/$tag/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:"$re" --launch-skip $skip --launch-count 1 \
    -o gpurun_out/$tag/one python tools/prof_run.py --config $cfg > gpurun_out/$tag/ncu.log 2>&1
ncu -i gpurun_out/$tag/one.ncu-rep --page raw --csv > gpurun_out/$tag/raw.csv 2>/dev/null
ncu -i gpurun_out/$tag/one.ncu-rep --page details > gpurun_out/$tag/details.txt 2>/dev/null
ncu -i gpurun_out/$tag/one.ncu-rep --page source --csv --print-source sass > gpurun_out/$tag/sass.csv 2>/dev/null
ls -la gpurun_out/$tag
