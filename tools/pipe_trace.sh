cd $GRAFT_REPO_ROOT
for v in "OZGPU_PIPE_PANELS=1,OZGPU_PIPE_LAST=1" "OZGPU_PIPE_PANELS=4" ; do
echo "=== $v"
env $(echo $v | tr ',' ' ') OZGPU_PIPE_TRACE=1 timeout 300 python tools/e2e_ab.py --steps 1 --rounds 1 "" 2>&1 | tail -40
done
nvidia-smi -q | grep -i -E "product name|link|pcie|gen|width" | head -20
