#!/bin/bash
O=gpurun_out/rows; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_spectral.py tests/test_gpu_algorithms.py tests/test_capi.py tests/test_gpu_guards.py -m gpu -q > $O/pytest.log 2>&1; tail -3 $O/pytest.log
for c in 2 7; do
  python bench.py --config $c --no-cpu --no-e2e --steps 5 --warmup 3 > $O/b$c.json 2> $O/b$c.err
  python -c "import json;d=json.load(open('$O/b$c.json'));print($c,d['ms_per_step'],d['volume_sha256_16'])"
done
PF_CFG=2 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/step_c2.csv python tools/prof_step.py > $O/step_c2.log 2>&1
python tools/launches.py $O/step_c2.csv > $O/step_c2.txt; head -8 $O/step_c2.txt
