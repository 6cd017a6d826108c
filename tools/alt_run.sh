#!/bin/bash
# Swap in an alternative build of libpbit.so (tools/alt/<name>.so) for one command.
set -e
lib=paper_cs_0511020_b200/libpbit.so
cp $lib /tmp/libpbit.keep.so
cp tools/alt/$1.so $lib
shift
"$@" || true
cp /tmp/libpbit.keep.so $lib
