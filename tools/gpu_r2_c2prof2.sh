#!/bin/bash
# Config-2 step launch list at HEAD (fused type-2 start, W = 17 readout, PFA 35-point DFTs)
O=gpurun_out/c2prof; mkdir -p $O
PF_CFG=2 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file $O/step_c2.csv python tools/prof_step.py > $O/step_c2.log 2>&1
python tools/launches.py $O/step_c2.csv | head -25
