#!/bin/bash
# exponential-of-semicircle window: NUFFT-related tests, configs 1/2/5/7 with both windows
O=gpurun_out/es; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_spectral.py tests/test_gpu_algorithms.py tests/test_capi.py tests/test_gpu_guards.py tests/test_gpu_acceptance.py tests/test_gpu_onchip.py tests/test_gpu_configs.py -m gpu -q > $O/pytest.log 2>&1; tail -15 $O/pytest.log
for wdw in es; do
for c in 2; do
  PF_NUFFT_WINDOW=$wdw python bench.py --config $c --no-cpu --no-e2e --steps 5 --warmup 3 > $O/bench_c${c}_$wdw.json 2> $O/bench_c${c}_$wdw.err
  python -c "import json;d=json.load(open('$O/bench_c${c}_$wdw.json'));print($c,'$wdw',d['ms_per_step'],d['volume_sha256_16'])"
done; done
PF_CFG=2 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/step_c2.csv python tools/prof_step.py > $O/step_c2.log 2>&1
python tools/launches.py $O/step_c2.csv > $O/step_c2.txt; head -8 $O/step_c2.txt
PF_CFG=7 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/step_c7.csv python tools/prof_step.py > $O/step_c7.log 2>&1
python tools/launches.py $O/step_c7.csv > $O/step_c7.txt; head -6 $O/step_c7.txt
PF_CFG=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/step_c1.csv python tools/prof_step.py > $O/step_c1.log 2>&1
python tools/launches.py $O/step_c1.csv > $O/step_c1.txt; head -6 $O/step_c1.txt
