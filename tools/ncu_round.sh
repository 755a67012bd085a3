# ncu --set full captures of the hot kernels with the current library (read back with ncu -i)
NCU="ncu --set full --import-source on --clock-control none -s 2 -c 1"
GE=gelu GN=8192 $NCU -k regex:gemm_bf16 -f -o gpurun_out/ncu_gelu python tools/gemm_one.py > gpurun_out/ncu_gelu.log 2>&1
GE=dgelu GN=8192 GBM=1 $NCU -k regex:gemm_bf16 -f -o gpurun_out/ncu_dgelu python tools/gemm_one.py > gpurun_out/ncu_dgelu.log 2>&1
GE=acc_f32 GM=6144 GN=2048 GK=16384 GAM=1 GBM=1 $NCU -k regex:gemm_bf16 -f -o gpurun_out/ncu_wgrad python tools/gemm_one.py > gpurun_out/ncu_wgrad.log 2>&1
GE=bf16 $NCU -k regex:gemm_bf16 -f -o gpurun_out/ncu_qkv python tools/gemm_one.py > gpurun_out/ncu_qkv.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:attn_bwd_tc64 -s 1 -c 1 -f -o gpurun_out/ncu_attn_bwd python tools/attn_one.py > gpurun_out/ncu_attn_bwd.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:attn_fwd_tc -s 1 -c 1 -f -o gpurun_out/ncu_attn_fwd python tools/attn_one.py > gpurun_out/ncu_attn_fwd.log 2>&1
