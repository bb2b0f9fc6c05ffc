#!/bin/bash
O=gpurun_out/g3; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_algorithms.py tests/test_gpu_acceptance.py tests/test_gpu_guards.py tests/test_gpu_edge.py -m gpu -q > $O/pytest.log 2>&1; tail -3 $O/pytest.log
for v in 1 0; do for c in 2 7; do
  PF_G3_EVEN=$v python bench.py --config $c --no-cpu --no-e2e --steps 5 --warmup 3 > $O/b.json 2> $O/b.err
  python -c "import json;d=json.load(open('$O/b.json'));print($c,'even',$v,d['ms_per_step'],d['volume_sha256_16'])"
done; done
PF_PARITY_LOG=$O/parity.jsonl timeout 900 python -m pytest tests/test_gpu_parity_full.py -m gpu -q -k "config2 or c2" > $O/pytest_full.log 2>&1; tail -2 $O/pytest_full.log; cat $O/parity.jsonl | cut -c1-160
