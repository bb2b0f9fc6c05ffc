#!/bin/bash
# ncu --set full of one type-2 readout launch at config 2: tiled vs per-point half-warp kernel.
O=gpurun_out/interp_ncu; mkdir -p $O
PF_CFG=2 ncu --set full --clock-control none --import-source on -k regex:"k_interp2" -s 4 -c 1 \
    -o $O/tiles python tools/prof_step.py > $O/tiles.log 2>&1
PF_INTERP_TILES=0 PF_CFG=2 ncu --set full --clock-control none --import-source on -k regex:"k_interp2" -s 4 -c 1 \
    -o $O/half python tools/prof_step.py > $O/half.log 2>&1
ls -la $O
