#!/bin/bash
# A/B: bounds-test-free staging / constant-trip write-out for full tiles
set -u
for cfg in C3 C4 C2; do
  echo "== $cfg"; bash tools/variant_run.sh $cfg fs0 fs1 fw1 fsw fs0 fsw
done
