#!/bin/bash
# A/B: pass-0 gather: segment position and slot in one round trip; segment-table L2 prefetch
set -u
for cfg in C3 C4 C2 C5; do
  echo "== $cfg"; bash tools/variant_run.sh $cfg g00 gp gm gpm g00 gpm
done
