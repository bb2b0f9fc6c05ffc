#!/bin/bash
O=gpurun_out/x2; mkdir -p $O
for x in large 10; do
for c in 2 7; do
  PF_XFFT=$x python bench.py --config $c --no-cpu --no-e2e --steps 5 --warmup 3 > $O/b.json 2> $O/b.err
  python -c "import json;d=json.load(open('$O/b.json'));print($c,'$x',d['ms_per_step'],d['volume_sha256_16'])"
done; done
