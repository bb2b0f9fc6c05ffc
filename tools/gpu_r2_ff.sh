#!/bin/bash
O=gpurun_out/ff; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_algorithms.py tests/test_gpu_guards.py tests/test_gpu_edge.py tests/test_gpu_acceptance.py tests/test_capi.py -m gpu -q > $O/pytest.log 2>&1; tail -3 $O/pytest.log
for v in 1 0; do
  PF_READOUT_FUSED=$v python bench.py --config 2 --no-cpu --no-e2e --steps 5 --warmup 3 > $O/b$v.json 2> $O/b$v.err
  python -c "import json;d=json.load(open('$O/b$v.json'));print(2,'fused',$v,d['ms_per_step'],d['volume_sha256_16'])"
done
PF_PARITY_LOG=$O/parity.jsonl timeout 900 python -m pytest tests/test_gpu_parity_full.py -m gpu -q -k "config2 or c2" > $O/pytest_full.log 2>&1; tail -2 $O/pytest_full.log; cat $O/parity.jsonl | cut -c1-160
PF_CFG=2 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/step_c2.csv python tools/prof_step.py > $O/step_c2.log 2>&1
python tools/launches.py $O/step_c2.csv > $O/step_c2.txt; head -7 $O/step_c2.txt
