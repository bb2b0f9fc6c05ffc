# config-3 (SRSD) launch list: 2 frequencies, all 128 planes (tools/prof_rsd.py)
mkdir -p gpurun_out/c3l
O=gpurun_out/c3l
PF_CFG=3 PF_NF=2 python tools/prof_rsd.py > $O/plain.log 2>&1 && \
PF_CFG=3 PF_NF=2 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv \
  --log-file $O/launches_c3.csv python tools/prof_rsd.py > $O/ncu.log 2>&1
python tools/launches.py $O/launches_c3.csv > $O/launches_c3.txt 2>&1; head -12 $O/launches_c3.txt
