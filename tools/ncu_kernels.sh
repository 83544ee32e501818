#!/bin/bash
# Per-kernel time / DRAM bytes / occupancy of one multiply (all kernels of the 3rd call).
# Usage: tools/ncu_kernels.sh <tag> [gemm_ab args]   (env variants via OZGPU_* in the environment)
TAG=$1; shift
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread
timeout 600 ncu --metrics $M --clock-control none -k regex:"slice|rowmax|colmax|combine" --csv \
  python tools/gemm_ab.py --steps 1 --rounds 1 "$@" 2>/dev/null | grep -E '^"[0-9]' | \
  awk -F'","' '{printf "%-40s %-32s %s\n", substr($5,1,40), $(NF-2), $NF}'
