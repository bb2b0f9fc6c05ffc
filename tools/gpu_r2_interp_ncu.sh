#!/bin/bash
# ncu --set full of the type-2 readout kernel in one config-2 step
O=gpurun_out/interp_ncu; mkdir -p $O
PF_CFG=2 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_interp2 -s 0 -c 1 \
   --profile-from-start off -o $O/interp python tools/prof_step.py > $O/ncu.log 2>&1
tail -2 $O/ncu.log
