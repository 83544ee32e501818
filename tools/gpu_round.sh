#!/bin/bash
# One GPU session: parity tests, bench line, ncu launch list + full capture of the pair GEMM.
# Usage: tools/gpu_round.sh <tag> [bench args...]
set -u
TAG=${1:-r01}; shift || true
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > $OUT/${TAG}_smi.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/${TAG}_pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/${TAG}_pytest_gpu.txt
tail -3 $OUT/${TAG}_pytest_gpu.txt
timeout 900 python bench.py "$@" > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err; echo "bench rc=$?"
cat $OUT/${TAG}_bench.json; tail -5 $OUT/${TAG}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep "$@" > /dev/null 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_i8 -s 2 -c 1 -o $OUT/${TAG}_gemm \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep "$@" > $OUT/${TAG}_ncu_full.log 2>&1; echo "ncu full rc=$?"
tail -3 $OUT/${TAG}_ncu_full.log
