#!/bin/bash
# Event timeline of the blocked host pipeline (ozgpu_dgemm) for env variants.
# Usage: tools/pipe_trace.sh "VAR=V,VAR=V" ...
cd ${GRAFT_REPO_ROOT:-.}
for v in "$@"; do
  echo "=== $v"
  env $(echo $v | tr ',' ' ') OZGPU_PIPE_TRACE=1 timeout 300 python tools/e2e_ab.py --steps 1 --rounds 1 "" 2>&1 | tail -40
done
