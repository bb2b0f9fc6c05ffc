#!/bin/bash
# lanes x batch sweep at config 4 with the fused B kernel
mkdir -p gpurun_out/sweep
O=gpurun_out/sweep
for ln in 2 3 4; do for cap in 2 4 8; do
  PF_LANES=$ln PF_BATCH_CAP=$cap python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > $O/b_${ln}_${cap}.json 2>/dev/null
  python -c "import json; d=json.load(open('$O/b_${ln}_${cap}.json')); print('lanes=$ln cap=$cap', round(d['ms_per_step'],3), round(d['stage_ms']['propagation'],3))" 2>/dev/null || echo "lanes=$ln cap=$cap fail"
done; done
