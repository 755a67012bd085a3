# Round-2 ncu evidence (run on the GPU box from the repo root; results in gpurun_out/):
#  1. launch list of the bench command itself (first 1300 launches = the warm-up's first micro-batches)
#  2. ncu --set full of the hot kernels: qkv GEMM (the roofline kernel), GELU / dGELU / wgrad GEMMs,
#     the LM-head GEMM with the fused CE epilogue, attention fwd / bwd, the aggregation kernel
#  3. raw csv exports folded into profiles/r02_ncu_summary.json by tools/ncu_summarize.py
set -x
ncu --metrics gpu__time_duration.sum --clock-control none -c 1300 --csv --log-file gpurun_out/r02_launches_bench_cmd.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_bench_cmd.log 2>&1
python tools/launch_summary.py gpurun_out/r02_launches_bench_cmd.csv embed_fwd_kernel 2 > gpurun_out/r02_launches_bench_cmd.txt
NCU="ncu --set full --import-source on --clock-control none -s 2 -c 1"
GE=bf16 $NCU -k regex:gemm_bf16 -f -o gpurun_out/ncu_qkv python tools/gemm_one.py > /dev/null 2>&1
GE=gelu GN=8192 $NCU -k regex:gemm_bf16 -f -o gpurun_out/ncu_gelu python tools/gemm_one.py > /dev/null 2>&1
GE=dgelu GN=8192 GBM=1 $NCU -k regex:gemm_bf16 -f -o gpurun_out/ncu_dgelu python tools/gemm_one.py > /dev/null 2>&1
GE=acc_f32 GM=6144 GN=2048 GK=16384 GAM=1 GBM=1 $NCU -k regex:gemm_bf16 -f -o gpurun_out/ncu_wgrad python tools/gemm_one.py > /dev/null 2>&1
GE=ce_exp GM=8192 GN=32000 GK=2048 $NCU -k regex:gemm_bf16 -f -o gpurun_out/ncu_lmhead_ce python tools/gemm_one.py > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:attn_bwd_tc64 -s 1 -c 1 -f -o gpurun_out/ncu_attn_bwd python tools/attn_one.py > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:attn_fwd_tc -s 1 -c 1 -f -o gpurun_out/ncu_attn_fwd python tools/attn_one.py > /dev/null 2>&1
for k in qkv gelu dgelu wgrad lmhead_ce attn_bwd attn_fwd; do
  ncu -i gpurun_out/ncu_$k.ncu-rep --page raw --csv > gpurun_out/ncu_${k}_raw.csv 2>/dev/null
done
python tools/ncu_summarize.py gemmqkv gpurun_out/ncu_qkv_raw.csv gemm_gelu gpurun_out/ncu_gelu_raw.csv \
  gemm_dgelu gpurun_out/ncu_dgelu_raw.csv gemm_wgrad gpurun_out/ncu_wgrad_raw.csv gemm_lmhead_ce gpurun_out/ncu_lmhead_ce_raw.csv \
  attn_bwd gpurun_out/ncu_attn_bwd_raw.csv attn_fwd gpurun_out/ncu_attn_fwd_raw.csv
cp profiles/r02_ncu_summary.json gpurun_out/r02_ncu_summary.json
# keep gpurun_out under its 64 MiB copy-back limit: the GEMM reports other than qkv stay as csv only
rm -f gpurun_out/ncu_gelu.ncu-rep gpurun_out/ncu_dgelu.ncu-rep gpurun_out/ncu_wgrad.ncu-rep gpurun_out/ncu_lmhead_ce.ncu-rep
rm -f gpurun_out/r02_launches_bench_cmd.csv
