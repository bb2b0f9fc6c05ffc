#!/bin/bash
# ncu --set full (source counters) of the on-chip P = 140 kernel in one config-1 step
O=gpurun_out/ocncu; mkdir -p $O
PF_CFG=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_prop_onchip -c 1 \
   -o $O/onchip python tools/prof_step.py > $O/ncu.log 2>&1
tail -3 $O/ncu.log; ls -la $O
