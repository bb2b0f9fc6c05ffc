#!/bin/bash
# On-chip P = 140 propagation: tests, config-1 bench (on-chip vs generic), launch list.
O=gpurun_out/onchip; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_onchip.py tests/test_gpu_configs.py -k "onchip or config1" -q -x > $O/pytest.log 2>&1; tail -15 $O/pytest.log
python bench.py --config 1 > $O/bench_c1.json 2> $O/bench_c1.err; cut -c1-260 $O/bench_c1.json
PF_ONCHIP=0 python bench.py --config 1 --no-cpu --no-e2e > $O/bench_c1_generic.json 2> $O/bench_c1_generic.err; cut -c1-260 $O/bench_c1_generic.json
for g in 1 2 4 8 16; do PF_ONCHIP_GROUPS=$g python bench.py --config 1 --no-cpu --no-e2e > $O/bench_c1_g$g.json 2>/dev/null; echo "groups $g: $(python -c "import json;d=json.load(open('$O/bench_c1_g$g.json'));print(d['ms_per_step'])")"; done
PF_CFG=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file $O/step_c1.csv python tools/prof_step.py > $O/step_c1.log 2>&1
PF_CFG=1 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_prop_onchip -c 1 \
   -o $O/onchip_full python tools/prof_step.py > $O/ncu_full.log 2>&1
ls $O
