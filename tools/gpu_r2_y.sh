#!/bin/bash
O=gpurun_out/y; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_algorithms.py tests/test_capi.py tests/test_gpu_guards.py tests/test_gpu_acceptance.py -m gpu -q > $O/pytest.log 2>&1; tail -3 $O/pytest.log
for c in 2 7; do
  python bench.py --config $c --no-cpu --no-e2e --steps 5 --warmup 3 > $O/b$c.json 2> $O/b$c.err
  python -c "import json;d=json.load(open('$O/b$c.json'));print($c,d['ms_per_step'],d['volume_sha256_16'])"
done
