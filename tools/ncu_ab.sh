#!/bin/bash
# DRAM / L2 / tensor metrics of the pair-GEMM kernel for several env variants
# (each captured REPS times, interleaved).  Usage: REPS=3 tools/ncu_ab.sh <tag> "VAR=V,VAR=V" ...
TAG=$1; shift
REPS=${REPS:-1}
N=${AB_N:-8192}
M=gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second
for r in $(seq $REPS); do
for v in "$@"; do
  echo "== rep $r: $v"
  env $(echo $v | tr ',' ' ') timeout 300 ncu --metrics $M --clock-control base -k regex:gemm_i8 -c 1 --csv \
    python tools/gemm_ab.py --n $N --steps 1 --rounds 1 "$v" 2>/dev/null | grep -E '"(gpu__time|dram__bytes|lts__t_sector|sm__pipe|sm__cycles)' | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
done
