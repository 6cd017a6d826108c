#!/bin/bash
# A/B: L2 prefetch of the slot ranges of a future tile in the gather pass (pass 0)
set -u
for cfg in C3 C4 C2; do
  echo "== $cfg"; bash tools/variant_run.sh $cfg g0 g37 g74 g148 g0
done
