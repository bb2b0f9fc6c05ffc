#!/bin/bash
O=gpurun_out/x; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_edge.py tests/test_gpu_spectral.py tests/test_capi.py -m gpu -q > $O/pytest.log 2>&1; tail -3 $O/pytest.log
python tools/c2_shapes.py 2 > $O/c2_shapes.txt 2>&1; tail -4 $O/c2_shapes.txt
for x in large all; do
  PF_XFFT=$x python bench.py --config 2 --no-cpu --no-e2e --steps 5 --warmup 3 > $O/bench_c2_$x.json 2> $O/bench_c2_$x.err
  python -c "import json;d=json.load(open('$O/bench_c2_$x.json'));print('$x',d['ms_per_step'],d['volume_sha256_16'])"
done
