#!/bin/bash
# Bench lines for every config + ncu (launch list and full sets of the pair GEMM,
# slicing and combine kernels) on the headline config.  Usage: tools/gpu_perf.sh <tag>
set -u
TAG=${1:-r02}
OUT=gpurun_out
mkdir -p $OUT
Q="--no-e2e --no-cpu-baseline --no-sweep --no-traffic --no-north-star"
timeout 900 python bench.py > $OUT/${TAG}_bench_c2.json 2> $OUT/${TAG}_bench_c2.err; echo "c2 rc=$?"
# c1 is ~50 us per multiply: enough steps that the event timing is not the noise
timeout 600 python bench.py --config c1 --steps 300 --warmup 10 --no-sweep > $OUT/${TAG}_bench_c1.json 2> $OUT/${TAG}_bench_c1.err; echo "c1 rc=$?"
for c in c3 c4 ns; do
  timeout 600 python bench.py --config $c --steps 5 --no-sweep > $OUT/${TAG}_bench_$c.json 2> $OUT/${TAG}_bench_$c.err; echo "$c rc=$?"
done
timeout 900 python bench.py --config c5 --steps 3 --warmup 3 --no-sweep > $OUT/${TAG}_bench_c5.json 2> $OUT/${TAG}_bench_c5.err; echo "c5 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 3 $Q > /dev/null 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_i8 -s 2 -c 1 -o $OUT/${TAG}_gemm \
  python bench.py --steps 1 --warmup 3 $Q > $OUT/${TAG}_ncu_gemm.log 2>&1; echo "ncu gemm rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"slice_|colmax|rowmax|combine" -s 8 -c 4 -o $OUT/${TAG}_aux \
  python bench.py --steps 1 --warmup 3 $Q > $OUT/${TAG}_ncu_aux.log 2>&1; echo "ncu aux rc=$?"
for f in $OUT/${TAG}_bench_*.json; do echo "== $f"; python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1])
print({k:d.get(k) for k in ('value','ms_per_step','int8_tops','stage_ms')}, d.get('config',{}).get('slices'), d.get('clocks',{}).get('sm_mhz'), (d.get('e2e') or {}).get('value'), (d.get('cpu_baseline') or {}).get('value'))
" 2>&1 | tail -1; done
