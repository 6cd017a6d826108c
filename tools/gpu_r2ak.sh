#!/bin/bash
# A/B: branch-free staging (scratch slots for items past the tile end); parity of the variant
set -u
for cfg in C3 C4 C2 C5; do
  echo "== $cfg"; bash tools/variant_run.sh $cfg ss0 ss1 ss0 ss1 | python -c "
import sys,re
for l in sys.stdin:
    m=re.match(r'(\S+): ([\d.]+) (.*)',l)
    print(l.strip() if not m else m.group(1)+' '+m.group(2)+' '+str({k:v for k,v in eval(m.group(3)).items() if k.startswith('pass')}))"
done
PBIT_LIB_PATH=build/var/libpbit_ss1.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
