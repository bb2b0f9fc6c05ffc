#!/bin/bash
# On-chip P = 140 v2 (prime-factor lines): tests (incl. every register-FFT length), config-1
# warps x groups sweep, config-2 bench (PFA 35 / 20 in its 700-point lines), ncu of the kernel.
O=gpurun_out/onchip2; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_onchip.py tests/test_gpu_rsd.py tests/test_gpu_configs.py -k "onchip or config1 or fft" -q -x > $O/pytest.log 2>&1; tail -3 $O/pytest.log
for w in 12 16; do for g in 0 4; do PF_ONCHIP_WARPS=$w PF_ONCHIP_GROUPS=$g python bench.py --config 1 --no-cpu --no-e2e > $O/c1_w${w}_g$g.json 2>$O/c1_w${w}_g$g.err; echo "warps $w groups $g: $(python -c "import json;d=json.load(open('$O/c1_w${w}_g$g.json'));print(d['ms_per_step'])")"; done; done
python bench.py --config 2 --no-cpu --no-e2e > $O/c2.json 2> $O/c2.err; echo "c2 $(python -c "import json;d=json.load(open('$O/c2.json'));print(d['ms_per_step'])")"
PF_CFG=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file $O/step_c1.csv python tools/prof_step.py > $O/step_c1.log 2>&1
PF_CFG=1 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_prop_onchip -c 1 \
   -o $O/onchip_full python tools/prof_step.py > $O/ncu_full.log 2>&1
ls $O
