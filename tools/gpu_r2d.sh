#!/bin/bash
set -u
mkdir -p gpurun_out/r2d
for cfg in C3 C2 C5; do bash tools/variant_run.sh $cfg main hist0 hist2 vec main; done
python tools/mg_one_rank.py C3
PBIT_MG_TRANSPORT=nccl python tools/mg_one_rank.py C3
python tools/mg_one_rank.py C5
