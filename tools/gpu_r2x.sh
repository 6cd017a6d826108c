#!/bin/bash
# A/B: L2 prefetch of the tile after next in the relink partition kernels
set -u
for cfg in C3 C4 C2; do
  echo "== $cfg"; bash tools/variant_run.sh $cfg pp0 pp1 pp0 pp1
done
