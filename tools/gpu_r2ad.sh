#!/bin/bash
# A/B: u32 warp counters (14 / 13 items per thread) vs u16 pairs (16), with the L2 prefetch
set -u
for cfg in C3 C4 C2; do
  echo "== $cfg"; bash tools/variant_run.sh $cfg main wc14 wc13 main
done
