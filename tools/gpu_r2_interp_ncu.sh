#!/bin/bash
# ncu --set full of one type-2 readout launch at config 2 (current default kernel).
O=gpurun_out/interp_ncu; mkdir -p $O
PF_CFG=2 ncu --set full --clock-control none --import-source on -k regex:"k_interp2" -s 4 -c 1 \
    -o $O/${1:-cur} python tools/prof_step.py > $O/${1:-cur}.log 2>&1
ls -la $O
