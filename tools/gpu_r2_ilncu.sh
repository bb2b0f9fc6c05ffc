#!/bin/bash
O=gpurun_out/ilncu; mkdir -p $O
PF_CFG=7 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_interp2 -s 1 -c 1 \
   --profile-from-start off -o $O/il python tools/prof_step.py > $O/ncu.log 2>&1
tail -1 $O/ncu.log
