#!/bin/bash
# config-2 step launch lists at several PF_FL_WANT (Stockham lines per CTA).
O=gpurun_out/c2want; mkdir -p $O
for k in 4 8 16 32; do
  PF_FL_WANT=$k PF_CFG=2 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/w$k.csv python tools/prof_step.py > /dev/null 2>&1
  python tools/launches.py $O/w$k.csv > $O/w$k.txt; echo "want $k"; grep "fft_lines\|interp" $O/w$k.txt
done
