# A/B of GEMM library variants: bash tools/ab_gemm.sh "name1 name2 ..." [GB_ONLY]
# "prod" = the in-tree libfedb200.so; others = tools/libfedb200_<name>.so
for rep in 1 2; do
  for v in $1; do
    if [ "$v" = prod ]; then lib=""; else lib="tools/libfedb200_$v.so"; fi
    FB_LIB_PATH=$lib GB_ONLY=${2:-fc_fwd_gelu,proj2_dgrad_dgelu,qkv_fwd,proj2_fwd_resid,fc_dgrad,qkv_wgrad} python tools/gemm_bench.py 2>&1 | sed "s/^/$v $rep /"
  done
done
