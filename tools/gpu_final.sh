#!/bin/bash
# Round-end evidence on one GPU: parity tests, smoke, the reference arm, every
# bench config, ncu launch list + full captures.  Usage: tools/gpu_final.sh <tag>
set -u
TAG=${1:-r02}
OUT=gpurun_out
mkdir -p $OUT
timeout 1500 python -m pytest tests -q -m gpu --durations=20 > $OUT/${TAG}_pytest_gpu.txt 2>&1; echo "pytest rc=$?" | tee -a $OUT/${TAG}_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/${TAG}_smoke.txt 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py --impl reference > $OUT/${TAG}_reference_arm.json 2> $OUT/${TAG}_reference_arm.err; echo "reference arm rc=$?"
bash tools/gpu_perf.sh $TAG
