#!/bin/bash
mkdir -p gpurun_out/heavy
O=gpurun_out/heavy
timeout 900 python -m pytest tests/test_gpu_rsd.py tests/test_gpu_guards.py -m gpu -q -x -k "horner or guards" > $O/pytest.log 2>&1; tail -3 $O/pytest.log
PF_PARITY_LOG=$O/parity_c6.jsonl timeout 900 python -m pytest tests/test_gpu_parity_full.py -m gpu -q -x -k config6 > $O/pytest_c6.log 2>&1; tail -3 $O/pytest_c6.log; cat $O/parity_c6.jsonl
python bench.py --config 6 --steps 3 --warmup 3 > $O/bench_c6.json 2> $O/bench_c6.err; python -c "
import json; d=json.load(open('$O/bench_c6.json')); print(d['ms_per_step'], d['stage_ms'], d['roofline']['frac'], d['roofline'].get('executed',{}).get('frac'), d['value'], d['e2e']['value'] if d['e2e'] else None, d['cpu_baseline']['value'])" || tail -5 $O/bench_c6.err
