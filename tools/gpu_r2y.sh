#!/bin/bash
# A/B: first lookback window loaded before the staging
set -u
for cfg in C3 C4 C2; do
  echo "== $cfg"; bash tools/variant_run.sh $cfg lb0 lb1 lb0 lb1
done
