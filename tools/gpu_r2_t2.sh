#!/bin/bash
# Fused type-2 start: bit-identity + algorithm parity + config 2 / 7 bench lines.
O=gpurun_out/t2; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_spectral.py tests/test_capi.py tests/test_gpu_algorithms.py -q -m gpu > $O/pytest.log 2>&1; tail -3 $O/pytest.log
timeout 900 python -m pytest tests/test_gpu_parity_full.py -q -m gpu -x -k "config2 or config7" > $O/parity.log 2>&1; tail -3 $O/parity.log
python bench.py --config 2 --no-cpu > $O/bench_c2.json 2> $O/bench_c2.err; tail -c 400 $O/bench_c2.json
python bench.py --config 7 --no-cpu --steps 3 --warmup 3 > $O/bench_c7.json 2> $O/bench_c7.err; tail -c 400 $O/bench_c7.json
PF_CFG=2 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/step_c2.csv python tools/prof_step.py > /dev/null 2>&1
python tools/launches.py $O/step_c2.csv > $O/step_c2.txt; head -12 $O/step_c2.txt
