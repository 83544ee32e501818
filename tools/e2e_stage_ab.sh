for v in "OZGPU_STAGE_OVERLAP=0" "OZGPU_STAGE_OVERLAP=1,OZGPU_STAGE_THREADS=16" "OZGPU_STAGE_OVERLAP=1,OZGPU_STAGE_THREADS=8" "OZGPU_STAGE_OVERLAP=1,OZGPU_STAGE_THREADS=12,OZGPU_PIPE_TRACE=1"; do
  env $(echo $v | tr ',' ' ') timeout 300 python -c "
import sys,time; sys.path.insert(0,'.')
import numpy as np, paper_2506_11277_b200 as oz
n=8192; a=oz.random_uniform(n,n,1,-.5,.5); b=oz.random_uniform(n,n,2,-.5,.5); c=np.empty((n,n))
cfg=oz.MmaConfig.int8_int32(); p=oz.make_plan(cfg,n,12,12)
oz.multiply(a,b,cfg,p,out=c)
ts=[]
for i in range(5):
    t=time.perf_counter(); oz.multiply(a,b,cfg,p,out=c); ts.append(time.perf_counter()-t)
print('$v', [round(x*1e3,1) for x in ts])
t=time.perf_counter(); x=np.empty_like(a); x[...]=a; print('numpy copy 512MiB ms', round((time.perf_counter()-t)*1e3,1))
" 2>&1 | grep -v "ozgpu pipe" ; done
