#!/bin/bash
mkdir -p gpurun_out/capi
O=gpurun_out/capi
timeout 900 python -m pytest tests/test_capi_rsd.py -q -x > $O/pytest.log 2>&1; tail -15 $O/pytest.log
PF_NF=16 PF_CFG=1 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv \
      --log-file $O/launches_c1.csv python tools/prof_rsd.py > $O/ncu_c1.log 2>&1
python tools/launches.py $O/launches_c1.csv | head -12
