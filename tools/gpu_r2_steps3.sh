#!/bin/bash
# one profiled step per configuration at HEAD (launch lists for the per-kernel roofline table)
O=gpurun_out/steps; mkdir -p $O
for c in 1 2 3 4 5 7; do
  PF_CFG=$c timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum \
     --clock-control none --csv --log-file $O/step_c$c.csv python tools/prof_step.py > $O/step_c$c.log 2>&1
  python tools/launches.py $O/step_c$c.csv > $O/step_c$c.txt
  tail -1 $O/step_c$c.log
done
python tools/kernel_roofline.py $O > $O/kernel_roofline.md; cat $O/kernel_roofline.md
