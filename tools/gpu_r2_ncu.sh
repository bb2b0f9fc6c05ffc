#!/bin/bash
# ncu --set full of the config-4 propagation kernels (A, fused B, C) + steady-state DRAM
# traffic of a whole 2-frequency run (application replay, no cache control)
mkdir -p gpurun_out/ncu2
O=gpurun_out/ncu2
PF_NF=2 python tools/prof_rsd.py > $O/plain.log 2>&1; cat $O/plain.log
PF_NF=2 timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"k_pa|k_pb12|k_pc_h" -s 6 -c 3 -o $O/prop_full \
    python tools/prof_rsd.py > $O/ncu_full.log 2>&1; tail -n 2 $O/ncu_full.log
PF_NF=2 timeout 1200 ncu --replay-mode application --cache-control none --clock-control none \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum \
    -k regex:"k_" --csv --log-file $O/traffic_app.csv python tools/prof_rsd.py > $O/ncu_app.log 2>&1
tail -n 3 $O/ncu_app.log; wc -l $O/traffic_app.csv
