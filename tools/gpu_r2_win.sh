#!/bin/bash
O=gpurun_out/win; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_spectral.py tests/test_gpu_algorithms.py tests/test_capi.py tests/test_gpu_guards.py tests/test_gpu_acceptance.py -m gpu -q > $O/pytest.log 2>&1; tail -4 $O/pytest.log
for wv in 1 0; do
for c in 2 7; do
  PF_T2_WINDOW=$wv python bench.py --config $c --no-cpu --no-e2e --steps 5 --warmup 3 > $O/bench_c${c}_w$wv.json 2> $O/bench_c${c}_w$wv.err
  python -c "import json;d=json.load(open('$O/bench_c${c}_w$wv.json'));print($c,$wv,d['ms_per_step'],d['volume_sha256_16'])"
done; done
