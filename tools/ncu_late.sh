# Late-round-2 ncu evidence for the kernels changed after the round-2 summary (run on the GPU box
# from the repo root; results in gpurun_out/): attention bwd (dh 128 and dh 64, ordered dQ), the
# warp LayerNorm backward, and the launch list of one fused C4 / C3 pass.
set -x
NCU="ncu --set full --import-source on --clock-control none"
$NCU -k regex:attn_bwd_tc64 -s 1 -c 1 -f -o gpurun_out/ncu_attn_bwd_late python tools/attn_one.py > /dev/null 2>&1
AO_H=12 AO_DH=64 $NCU -k regex:attn_bwd_tcd64 -s 1 -c 1 -f -o gpurun_out/ncu_attn_bwd64_late python tools/attn_one.py > /dev/null 2>&1
$NCU -k regex:ln_bwd_warp -s 2 -c 1 -f -o gpurun_out/ncu_ln_bwd_warp_late python tools/ln_bench.py > /dev/null 2>&1
for k in attn_bwd_late attn_bwd64_late ln_bwd_warp_late; do
  ncu -i gpurun_out/ncu_$k.ncu-rep --page raw --csv > gpurun_out/ncu_${k}_raw.csv 2>/dev/null
done
NCU_SUMMARY=r02_ncu_summary_late.json python tools/ncu_summarize.py attn_bwd_dh128 gpurun_out/ncu_attn_bwd_late_raw.csv \
  attn_bwd_dh64 gpurun_out/ncu_attn_bwd64_late_raw.csv ln_bwd_warp gpurun_out/ncu_ln_bwd_warp_late_raw.csv
cp profiles/r02_ncu_summary_late.json gpurun_out/
PM_B=16 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4_launches.csv python tools/profile_micro.py --config c4 --iters 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/c4_launches.csv embed_fwd_kernel 2 > gpurun_out/r02_launches_c4_fused_pass_late.txt
rm -f gpurun_out/*.csv gpurun_out/ncu_attn_bwd64_late.ncu-rep gpurun_out/ncu_ln_bwd_warp_late.ncu-rep
