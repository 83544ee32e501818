cd $GRAFT_REPO_ROOT
M=gpu__time_duration.sum,dram__bytes_read.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
for s in "4 4" "6 6" "12 12"; do
for v in "OZGPU_CTA_PAIR=1,OZGPU_PAIR_STAGES=4" "OZGPU_CTA_PAIR=1,OZGPU_PAIR_STAGES=5"; do
  echo "== s=$s $v"
  env $(echo $v | tr ',' ' ') timeout 300 ncu --metrics $M --clock-control base -k regex:gemm_i8 -c 1 --csv \
    python tools/gemm_ab.py --n 8192 --s $s --steps 1 --rounds 1 "" 2>/dev/null | grep -E '"(gpu__time|dram__bytes|sm__pipe)' | awk -F'","' '{print $(NF-2), $NF}'
done; done
