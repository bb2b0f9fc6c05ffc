#!/bin/bash
mkdir -p gpurun_out/sweep2
O=gpurun_out/sweep2
for c in 3 5 1; do for ln in 2 3 4; do
  PF_LANES=$ln python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e > $O/b_c${c}_${ln}.json 2>/dev/null
  python -c "import json; d=json.load(open('$O/b_c${c}_${ln}.json')); print('c$c lanes=$ln', round(d['ms_per_step'],3), round(d['stage_ms']['propagation'],3))" 2>/dev/null || echo "c$c lanes=$ln fail"
done; done
