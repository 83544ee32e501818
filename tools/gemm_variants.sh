#!/bin/bash
# Sustained (power-capped) interleaved timing + ncu DRAM/L2/tensor metrics of GEMM-path variants.
# Usage: [REPS=2] [AB_N=8192] tools/gemm_variants.sh <tag> "VAR=V,VAR=V" ...
TAG=$1; shift
OUT=gpurun_out
mkdir -p $OUT
N=${AB_N:-8192}
timeout 900 python tools/gemm_ab.py --n $N --steps ${AB_STEPS:-10} --rounds ${AB_ROUNDS:-3} "$@" > $OUT/${TAG}_ab.jsonl 2> $OUT/${TAG}_ab.err
cat $OUT/${TAG}_ab.jsonl
REPS=${REPS:-2} timeout 1200 bash tools/ncu_ab.sh $TAG "$@" > $OUT/${TAG}_ncu_ab.txt 2>&1
cat $OUT/${TAG}_ncu_ab.txt
