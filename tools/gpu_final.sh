#!/bin/bash
# Round-end evidence on one GPU: parity tests, smoke, every bench config, the
# reference arm, ncu launch list + full captures.  Usage: tools/gpu_final.sh <tag>
set -u
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
timeout 1500 python -m pytest tests -q -m gpu > $OUT/${TAG}_pytest_gpu.txt 2>&1; echo "pytest rc=$?" | tee -a $OUT/${TAG}_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/${TAG}_smoke.txt 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py --impl reference > $OUT/${TAG}_reference_arm.json 2> $OUT/${TAG}_reference_arm.err; echo "reference arm rc=$?"
timeout 900 python bench.py --config c5 --steps 3 --warmup 3 --no-sweep > $OUT/${TAG}_bench_c5.json 2> $OUT/${TAG}_bench_c5.err; echo "c5 rc=$?"
bash tools/gpu_perf.sh $TAG
