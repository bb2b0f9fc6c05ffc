#!/bin/bash
# 16 x 16 trimmed readout: tests, config 2 / 7 bench lines with both modes
O=gpurun_out/trim; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_algorithms.py -m gpu -q > $O/pytest.log 2>&1; tail -3 $O/pytest.log
for v in "2 4" "2 8" "1 4"; do
set -- $v
for c in 2 7; do
  PF_INTERP_H17=$1 PF_INTERP_UNROLL=$2 python bench.py --config $c --no-cpu --no-e2e --steps 5 --warmup 3 > $O/bench_c${c}_m$1$2.json 2> $O/bench_c${c}_m$1$2.err
  python -c "import json;d=json.load(open('$O/bench_c${c}_m$1$2.json'));print($c,$1,$2,d['ms_per_step'],d['volume_sha256_16'])"
done; done
