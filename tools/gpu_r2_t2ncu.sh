#!/bin/bash
O=gpurun_out/t2ncu; mkdir -p $O
PF_CFG=2 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_t2_ -s 2 -c 2 \
   --profile-from-start off -o $O/t2 python tools/prof_step.py > $O/ncu.log 2>&1
tail -2 $O/ncu.log
