#!/bin/bash
mkdir -p gpurun_out/xfft2
O=gpurun_out/xfft2
timeout 1500 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_parity_full.py > $O/pytest_all.log 2>&1; tail -3 $O/pytest_all.log
PF_PARITY_LOG=$O/parity.jsonl timeout 600 python -m pytest tests/test_gpu_configs.py -m gpu -q -x -k "config1 or config0" > $O/pytest_c1.log 2>&1; tail -2 $O/pytest_c1.log; cat $O/parity.jsonl
for x in 0 1; do for c in 1 2; do
PF_XFFT=$x python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e > $O/b_c${c}_x$x.json 2>/dev/null
python -c "import json; d=json.load(open('$O/b_c${c}_x$x.json')); print('xfft=$x c$c', round(d['ms_per_step'],3), round(d['stage_ms']['propagation'],3))"
done; done
PF_NF=16 PF_CFG=1 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv \
      --log-file $O/launches_c1.csv python tools/prof_rsd.py > /dev/null 2>&1
python tools/launches.py $O/launches_c1.csv 2>&1 | head -8
