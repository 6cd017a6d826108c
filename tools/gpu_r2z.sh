#!/bin/bash
# A/B: pass kernel 1024-thread CTAs (16K-item tiles, 1 CTA/SM) vs 512 (8K, 2 CTAs/SM)
set -u
for cfg in C3 C4 C2 C5; do
  echo "== $cfg"; bash tools/variant_run.sh $cfg main t1024 main t1024
done
