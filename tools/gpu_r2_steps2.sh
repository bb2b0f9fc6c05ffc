#!/bin/bash
# one profiled step for configs 1, 2, 3, 7 at HEAD (launch lists)
O=gpurun_out/steps2; mkdir -p $O
for c in 1 2 3 7; do
  PF_CFG=$c timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum \
     --clock-control none --csv --log-file $O/step_c$c.csv python tools/prof_step.py > $O/step_c$c.log 2>&1
  python tools/launches.py $O/step_c$c.csv > $O/step_c$c.txt; head -12 $O/step_c$c.txt
done
