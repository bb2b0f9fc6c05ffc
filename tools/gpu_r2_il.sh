#!/bin/bash
O=gpurun_out/il; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_algorithms.py tests/test_gpu_guards.py -m gpu -q -k "voxel or cloud or zcheb or guard" > $O/pytest.log 2>&1; tail -3 $O/pytest.log
for v in 1 0; do
  PF_ZCHEB_IL=$v python bench.py --config 7 --no-cpu --no-e2e --steps 5 --warmup 3 > $O/b$v.json 2> $O/b$v.err
  python -c "import json;d=json.load(open('$O/b$v.json'));print(7,'il',$v,d['ms_per_step'],d['volume_sha256_16'])"
done



