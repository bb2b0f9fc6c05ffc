#!/bin/bash
# Round 2: smoke, full-size parity (configs 2/3/4/5 over whole volumes), bench --gpus 2 (gloo on one GPU)
mkdir -p gpurun_out/r2p
O=gpurun_out/r2p
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -2 $O/smoke.log
PF_PARITY_LOG=$O/parity_full.jsonl timeout 2400 python -m pytest tests/test_gpu_parity_full.py -m gpu -q -x --durations=0 > $O/pytest_full.log 2>&1; tail -12 $O/pytest_full.log
cat $O/parity_full.jsonl
python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_n1.json 2> $O/bench_n1.err
PF_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_n2.json 2> $O/bench_n2.err
python -c "
import json
for n in (1,2):
    try:
        d=json.loads(open('$O/bench_n%d.json'%n).read().strip().splitlines()[-1]); print(n, d['n_gpus'], d['ms_per_step'], d['volume_sha256_16'], d.get('dist_backend'))
    except Exception as e: print(n, 'fail', e)
"
tail -5 $O/bench_n2.err
