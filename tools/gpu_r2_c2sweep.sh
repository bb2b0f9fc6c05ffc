#!/bin/bash
mkdir -p gpurun_out/c2s
for mb in 16 32 64 128 256; do
  PF_READOUT_MB=$mb python bench.py --config 2 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/c2s/b_$mb.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/c2s/b_$mb.json')); print('readout_mb=$mb', round(d['ms_per_step'],3))" || echo fail $mb
done
