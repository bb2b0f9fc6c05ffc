#!/bin/bash
for cfg in "64 2 8" "32 4 8" "16 6 8" "32 4 12" "64 4 16" "128 3 8"; do
  set -- $cfg
  PF_STAGE_MB=$1 PF_STAGE_BUFS=$2 PF_STAGE_THREADS=$3 python - <<PY
import os, sys, time, torch, numpy as np
sys.path.insert(0, ".")
import paper_2501_05244_b200 as pf
from paper_2501_05244_b200 import configs
cfg = configs.config(4); k = configs.kernel(cfg)
h = configs.transients(cfg, device=torch.device("cuda")).cpu().numpy()
m = pf.TransientMeasurement(cfg.relay, cfg.illuminations, h, cfg.delta_t, cfg.t0)
pf.to_frequency(m, k); torch.cuda.synchronize()
ts = []
for _ in range(3):
    t = time.perf_counter(); pf.to_frequency(m, k); torch.cuda.synchronize(); ts.append(time.perf_counter() - t)
print("stage MB=$1 bufs=$2 threads=$3: to_frequency %.1f ms" % (min(ts) * 1e3))
PY
done
