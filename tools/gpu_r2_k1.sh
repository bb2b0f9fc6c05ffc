#!/bin/bash
O=gpurun_out/k1; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_rsd.py tests/test_gpu_guards.py -m gpu -q -k "k1 or K1 or temporal or to_frequency or guard" > $O/pytest.log 2>&1; tail -3 $O/pytest.log
python tools/k1_ab.py | tee $O/k1_c4.json
PF_CFG=3 python tools/k1_ab.py | tee $O/k1_c3.json
python bench.py --no-cpu --no-e2e --steps 5 --warmup 3 > $O/bench_c4.json 2> $O/bench_c4.err
python -c "import json;d=json.load(open('$O/bench_c4.json'));print(d['ms_per_step'],d['stage_ms'],d['roofline_other']['frac'])"
