#!/bin/bash
# one profiled step per configuration: kernel launch lists for the per-kernel roofline table
mkdir -p gpurun_out/steps
O=gpurun_out/steps
for c in 0 1 2 3 4 5; do
  PF_CFG=$c timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum \
     --clock-control none --csv --log-file $O/step_c$c.csv python tools/prof_step.py > $O/step_c$c.log 2>&1
  tail -1 $O/step_c$c.log
done
