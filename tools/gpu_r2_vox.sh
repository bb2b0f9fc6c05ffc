#!/bin/bash
mkdir -p gpurun_out/vox
O=gpurun_out/vox
timeout 900 python -m pytest tests/test_gpu_algorithms.py -q -x -k "voxel" > $O/pytest.log 2>&1; tail -3 $O/pytest.log
PF_PARITY_LOG=$O/parity.jsonl timeout 1200 python -m pytest tests/test_gpu_parity_full.py -q -x -k "config7" > $O/pytest_c7.log 2>&1; tail -3 $O/pytest_c7.log; cat $O/parity.jsonl
python bench.py --config 7 --steps 3 --warmup 3 --no-e2e > $O/bench_c7.json 2> $O/bench_c7.err; python -c "
import json; d=json.load(open('$O/bench_c7.json')); print(d['ms_per_step'], d['value'], d['stage_ms'], d['roofline']['frac'], d['cpu_baseline'])" || tail -5 $O/bench_c7.err
PF_CFG=7 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/step_c7.csv python tools/prof_step.py > /dev/null 2>&1
python tools/launches.py $O/step_c7.csv | head -10
