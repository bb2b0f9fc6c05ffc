#!/bin/bash
O=gpurun_out/skip; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_spectral.py tests/test_gpu_algorithms.py tests/test_capi.py tests/test_gpu_guards.py tests/test_gpu_acceptance.py tests/test_gpu_configs.py tests/test_gpu_edge.py -m gpu -q > $O/pytest.log 2>&1; tail -4 $O/pytest.log
for sk in 1 0; do
for c in 1 2 7; do
  PF_T1_SKIP_ZERO=$sk python bench.py --config $c --no-cpu --no-e2e --steps 5 --warmup 3 > $O/bench_c${c}_s$sk.json 2> $O/bench_c${c}_s$sk.err
  python -c "import json;d=json.load(open('$O/bench_c${c}_s$sk.json'));print($c,$sk,d['ms_per_step'],d['volume_sha256_16'])"
done; done
