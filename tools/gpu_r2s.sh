#!/bin/bash
# ncu --set full + SASS source of pass 1 and pass 0 (C3), for the pass instruction budget
set -u
bash tools/ncu_one.sh k_onesweep 1 os1
bash tools/ncu_one.sh k_onesweep 0 os0
