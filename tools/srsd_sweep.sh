#!/bin/bash
# SRSD (config 3) plane-batch / lane sweep: device ms per step
for v in "64 8 2" "64 8 3" "128 8 2" "128 8 3" "256 8 2" "64 4 2"; do
  set -- $v
  PF_SRSD_BATCH_MB=$1 PF_SRSD_MINQ=$2 PF_LANES=$3 python bench.py --config 3 --no-cpu --no-e2e > gpurun_out/sw.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/sw.json')); print('batchMB=$1 minq=$2 lanes=$3', round(d['ms_per_step'],3))"
done
