#!/bin/bash
# split type-2 start: tests, config 2 / 7 bench lines with and without
O=gpurun_out/split; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_spectral.py tests/test_gpu_algorithms.py tests/test_capi.py tests/test_gpu_guards.py -m gpu -q > $O/pytest.log 2>&1; tail -5 $O/pytest.log
for s in 1 0; do
for c in 2 7; do
  PF_T2_SPLIT=$s python bench.py --config $c --no-cpu --no-e2e --steps 5 --warmup 3 > $O/bench_c${c}_s$s.json 2> $O/bench_c${c}_s$s.err
  python -c "import json;d=json.load(open('$O/bench_c${c}_s$s.json'));print($c,$s,d['ms_per_step'],d['volume_sha256_16'])"
done; done
PF_CFG=2 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/step_c2.csv python tools/prof_step.py > $O/step_c2.log 2>&1
python tools/launches.py $O/step_c2.csv > $O/step_c2.txt; head -8 $O/step_c2.txt
