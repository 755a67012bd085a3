# ncu launch list of one C4 micro-batch fwd+bwd (the 2nd of 3), summarised per kernel
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_step.csv python tools/profile_micro.py --iters 2 > gpurun_out/launches_step.log 2>&1
python tools/launch_summary.py gpurun_out/launches_step.csv embed_fwd_kernel 2 > gpurun_out/launches_step_summary.txt
