#!/bin/bash
# One profiled config-2 step (launch list), plus the same with PF_INTERP_H17=0.
O=gpurun_out/c2step; mkdir -p $O
PF_CFG=2 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/a.csv python tools/prof_step.py > /dev/null 2>&1
PF_INTERP_H17=0 PF_CFG=2 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/b.csv python tools/prof_step.py > /dev/null 2>&1
python tools/launches.py $O/a.csv > $O/a.txt; python tools/launches.py $O/b.csv > $O/b.txt; grep interp $O/a.txt $O/b.txt
