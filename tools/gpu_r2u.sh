#!/bin/bash
# A/B: L2 prefetch of a tile one resident wave ahead in the pass kernel
set -u
for cfg in C3 C4 C2; do
  echo "== $cfg"; bash tools/variant_run.sh $cfg main pf148 pf296 pf592 main
done
