#!/bin/bash
# A/B: relink level 1 + apply per group of level-0 bins on device buffers (L2 reuse of the
# level-1 output), with / without discarding the applied records' L2 lines, with / without
# streaming stores in the partition
set -u
r() { bash tools/variant_run.sh C3 "$@" | python -c "
import sys,re
for l in sys.stdin:
    m=re.match(r'(\S+): ([\d.]+) (.*)',l)
    print(l.strip() if not m else m.group(1)+' '+m.group(2)+' relink '+str(eval(m.group(3)).get('relink')))"; }
r dc0 dc0:PBIT_RELINK_GROUPS=8 dc0:PBIT_RELINK_GROUPS=16 dc0:PBIT_RELINK_GROUPS=32 dc0:PBIT_RELINK_GROUPS=64
r dc1:PBIT_RELINK_GROUPS=8 dc1:PBIT_RELINK_GROUPS=16 dc1:PBIT_RELINK_GROUPS=32 dc1:PBIT_RELINK_GROUPS=64
r dc0s:PBIT_RELINK_GROUPS=16 dc0s:PBIT_RELINK_GROUPS=32 dc1s:PBIT_RELINK_GROUPS=16 dc1s:PBIT_RELINK_GROUPS=32 dc1s:PBIT_RELINK_GROUPS=64 dc0
