#!/bin/bash
O=gpurun_out/es2; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_algorithms.py tests/test_gpu_guards.py -m gpu -q > $O/pytest.log 2>&1; tail -2 $O/pytest.log
for u in 8 4; do
for c in 2 7; do
  PF_INTERP_UNROLL=$u python bench.py --config $c --no-cpu --no-e2e --steps 5 --warmup 3 > $O/bench_c${c}_u$u.json 2> $O/bench_c${c}_u$u.err
  python -c "import json;d=json.load(open('$O/bench_c${c}_u$u.json'));print($c,$u,d['ms_per_step'],d['volume_sha256_16'])"
done; done
