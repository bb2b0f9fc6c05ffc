#!/bin/bash
mkdir -p gpurun_out/dropin
O=gpurun_out/dropin
timeout 1500 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_parity_full.py > $O/pytest.log 2>&1; tail -3 $O/pytest.log
python bench.py --no-cpu > $O/bench_c4.json 2> $O/bench_c4.err; python -c "
import json; d=json.load(open('$O/bench_c4.json')); print(d['ms_per_step'], d['stage_ms'], d['e2e']['ms_per_step'], json.dumps(d['e2e_dropin']))" || tail -5 $O/bench_c4.err
