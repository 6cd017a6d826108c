#!/bin/bash
# Launch list (time + DRAM bytes) of selected kernels of one C3 call: tools/ncu_kernels.sh <regex> [config] [tag]
set -u
re=$1; cfg=${2:-C3}; tag=${3:-k}
mkdir -p gpurun_out
python tools/prof_run.py --config $cfg > gpurun_out/plain_$tag.log 2>&1 || { echo "plain run failed"; cat gpurun_out/plain_$tag.log; exit 1; }
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none \
    -k regex:"$re" --csv --log-file gpurun_out/ncu_$tag.csv python tools/prof_run.py --config $cfg > /dev/null 2>&1
python tools/ncu_table.py gpurun_out/ncu_$tag.csv
