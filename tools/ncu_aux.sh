#!/bin/bash
# Full-set ncu captures of the HBM-bound kernels (slicing, combine) on the headline config.
# Usage: tools/ncu_aux.sh <tag> [bench args]
TAG=$1; shift
OUT=gpurun_out
mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"slice_|rowmax|colmax|combine" -s 6 -c 5 -o $OUT/${TAG}_aux \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep "$@" > $OUT/${TAG}_ncu_aux.log 2>&1; echo "ncu aux rc=$?"
tail -3 $OUT/${TAG}_ncu_aux.log
