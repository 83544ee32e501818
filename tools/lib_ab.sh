#!/bin/bash
# A/B of two builds of libozgpu.so (e.g. a kernel rewrite against the
# previous build kept under tools/ablib/): per-stage device times from
# tools/slice_ab.py, alternating the libraries across rounds.
# Usage: tools/lib_ab.sh <base.so> [slice_ab args]
BASE=$1; shift
for r in 1 2 3; do
  for lib in "$BASE" default; do
    if [ "$lib" = default ]; then
      echo -n "new  r$r "; python tools/slice_ab.py "$@" | head -1
    else
      echo -n "base r$r "; OZGPU_LIB_OVERRIDE=$lib python tools/slice_ab.py "$@" | head -1
    fi
  done
done
