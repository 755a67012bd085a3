# raster group height sweep (FB_GEMM_GROUP_M overrides the 2-SM raster group for every GEMM)
for g in 16 2 3 4 5 6 8 16; do
  FB_GEMM_GROUP_M=$g GB_ONLY=qkv_fwd,fc_fwd_gelu,proj2_fwd_resid,proj2_dgrad_dgelu,fc_dgrad,qkv_wgrad,head_fwd python tools/gemm_bench.py | python -c "
import json,sys
print('G=$g', ' '.join(f\"{d['gemm']}={d['tflops_2sm']}\" + (f\"/{d['tflops_splitk_auto']}\" if 'tflops_splitk_auto' in d else '') for d in map(json.loads, sys.stdin)))"
done
