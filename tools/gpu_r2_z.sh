#!/bin/bash
O=gpurun_out/z; mkdir -p $O
for v in 0 1; do for c in 2 7; do
  PF_PROP_COLS_XL=$v python bench.py --config $c --no-cpu --no-e2e --steps 5 --warmup 3 > $O/b.json 2> $O/b.err
  python -c "import json;d=json.load(open('$O/b.json'));print($c,'cols_xl',$v,d['ms_per_step'],d['volume_sha256_16'])"
done; done
