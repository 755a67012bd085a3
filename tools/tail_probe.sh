GB_ONLY=qkv_wgrad,proj_wgrad python tools/gemm_bench.py
GE=acc_f32 GM=6144 GN=2048 GK=16384 GAM=1 GBM=1 python - <<'PY'
import os,sys,torch
sys.path.insert(0,'.')
from paper_2405_10853_b200 import ext
ext.lib()
M,N,K=6144,2048,16384
A=torch.randn(K,M,device='cuda').to(torch.bfloat16); B=torch.randn(K,N,device='cuda').to(torch.bfloat16)
C=torch.zeros(M,N,device='cuda'); ws=torch.empty(16<<20,device='cuda')
for i in range(3):
    ext.call("fb_gemm_bf16_splitk", M,N,K,A.data_ptr(),M,1,B.data_ptr(),N,1,C.data_ptr(),N,2,0,ws.data_ptr(),ws.numel()*4,ext.stream_handle())
torch.cuda.synchronize(); print("ok")
PY
ncu --set full --import-source on -k regex:gemm_bf16 -s 2 -c 1 -f -o gpurun_out/ncu_tailsplit python -c "
import sys,torch; sys.path.insert(0,'.')
from paper_2405_10853_b200 import ext
ext.lib()
M,N,K=6144,2048,16384
A=torch.randn(K,M,device='cuda').to(torch.bfloat16); B=torch.randn(K,N,device='cuda').to(torch.bfloat16)
C=torch.zeros(M,N,device='cuda'); ws=torch.empty(16<<20,device='cuda')
for i in range(3):
    ext.call('fb_gemm_bf16_splitk', M,N,K,A.data_ptr(),M,1,B.data_ptr(),N,1,C.data_ptr(),N,2,0,ws.data_ptr(),ws.numel()*4,ext.stream_handle())
torch.cuda.synchronize()
" > gpurun_out/ncu_tailsplit.log 2>&1
