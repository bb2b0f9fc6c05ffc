"""Short config-2 run for profiling (2 iterations)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_05244_b200 as pf  # noqa: E402
from paper_2501_05244_b200 import configs  # noqa: E402
from paper_2501_05244_b200.algorithms import nursd3d_explicit  # noqa: E402

cfg = configs.config(2)
hist = configs.transients(cfg, device=torch.device("cuda"))
k = pf.build_kernel(cfg.lambda_c, cfg.n_bins, cfg.delta_t)
for _ in range(2):
    coeff = pf.to_frequency_device(hist, k, cfg.t0)
    sl = pf.DeviceFrequencySlices(k.frequencies, coeff, cfg.relay, cfg.illuminations)
    vol = nursd3d_explicit(sl, cfg.grid, cfg.lattice)
torch.cuda.synchronize()
print("ok")
