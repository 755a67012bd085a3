set -x
python tools/gemm_bench.py > gpurun_out/gemm_bench.jsonl 2>&1
NCU="ncu --set full --import-source on --clock-control none -k regex:gemm_bf16 -s 2 -c 1"
GE=gelu GN=8192 $NCU -f -o gpurun_out/ncu_gelu python tools/gemm_one.py > gpurun_out/ncu_gelu.log 2>&1
GE=dgelu GN=8192 GBM=1 $NCU -f -o gpurun_out/ncu_dgelu python tools/gemm_one.py > gpurun_out/ncu_dgelu.log 2>&1
GE=acc_f32 GM=6144 GN=2048 GK=16384 GAM=1 GBM=1 $NCU -f -o gpurun_out/ncu_wgrad python tools/gemm_one.py > gpurun_out/ncu_wgrad.log 2>&1
GE=resid_f32 GN=2048 GK=8192 $NCU -f -o gpurun_out/ncu_resid python tools/gemm_one.py > gpurun_out/ncu_resid.log 2>&1
