#!/bin/bash
O=gpurun_out/c7; mkdir -p $O
PF_CFG=7 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/step_c7.csv python tools/prof_step.py > $O/step_c7.log 2>&1
python tools/launches.py $O/step_c7.csv > $O/step_c7.txt; head -10 $O/step_c7.txt
PF_CFG=3 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/step_c3.csv python tools/prof_step.py > $O/step_c3.log 2>&1
python tools/launches.py $O/step_c3.csv > $O/step_c3.txt; head -8 $O/step_c3.txt
