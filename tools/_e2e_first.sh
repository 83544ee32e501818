set -u
mkdir -p gpurun_out
OLD=OZGPU_PIPE_FIRST=1,OZGPU_PIPE_LAST=2
timeout 400 python tools/e2e_ab.py --n 8192 --s 12 12 --steps 4 --rounds 4 "" $OLD > gpurun_out/first2_c2.txt 2>&1; echo "c2 rc=$?"
timeout 400 python tools/e2e_ab.py --n 4096 --s 16 17 --steps 4 --rounds 4 "" $OLD OZGPU_PIPE=0 > gpurun_out/first2_c3.txt 2>&1; echo "c3 rc=$?"
timeout 300 python tools/e2e_ab.py --m 65536 --n 2048 --s 12 11 --steps 4 --rounds 4 "" $OLD > gpurun_out/first2_c4.txt 2>&1; echo "c4 rc=$?"
timeout 400 python tools/e2e_ab.py --n 16384 --s 13 12 --steps 2 --rounds 2 "" $OLD > gpurun_out/first2_ns.txt 2>&1; echo "ns rc=$?"
timeout 600 python -m pytest tests -x -q -m gpu -k "pipeline or large_shape or host" > gpurun_out/first2_pytest.txt 2>&1; echo "pytest rc=$?"
