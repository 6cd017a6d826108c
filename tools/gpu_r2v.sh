#!/bin/bash
# A/B: pass-kernel L2 prefetch distance sweep
set -u
for cfg in C3 C4; do
  echo "== $cfg"; bash tools/variant_run.sh $cfg main pf37 pf74 pf110 pf148 pf200 main
done
