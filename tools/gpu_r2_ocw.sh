#!/bin/bash
# on-chip P = 140 kernel: warps per CTA sweep on config 1
O=gpurun_out/ocw; mkdir -p $O
for w in 12 10 9 8; do
  PF_ONCHIP_WARPS=$w python bench.py --config 1 --no-cpu --no-e2e --steps 10 --warmup 3 > $O/bench_c1_w$w.json 2> $O/bench_c1_w$w.err
  python -c "import json;d=json.load(open('$O/bench_c1_w$w.json'));print($w,d['ms_per_step'],d['stage_ms']['propagation'],d['volume_sha256_16'])"
done
