"""Time BASELINE config 2 (non-planar relay -> 1e6 arbitrary voxels) on one GPU."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_05244_b200 as pf  # noqa: E402
from paper_2501_05244_b200 import configs  # noqa: E402
from paper_2501_05244_b200.algorithms import nursd3d_explicit  # noqa: E402

cfg = configs.config(2)
hist = configs.transients(cfg, device=torch.device("cuda"))
k = pf.build_kernel(cfg.lambda_c, cfg.n_bins, cfg.delta_t)
times = []
for it in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    coeff = pf.to_frequency_device(hist, k, cfg.t0)
    sl = pf.DeviceFrequencySlices(k.frequencies, coeff, cfg.relay, cfg.illuminations)
    vol = nursd3d_explicit(sl, cfg.grid, cfg.lattice)
    torch.cuda.synchronize()
    times.append(time.perf_counter() - t)
best = min(times[1:])
print(json.dumps({"config": "config2-nursd3d-explicit", "voxels": cfg.grid.count,
                  "n_freq": k.n_freq, "seconds": best, "voxels_per_s": cfg.grid.count / best,
                  "note": "wall clock incl. host planning (NUFFT plans, tile buckets) and D2H"}))
