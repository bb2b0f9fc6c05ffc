"""K1 alone on the config-$PF_CFG capture: median device time of 20 launches, HBM fraction."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_05244_b200 as pf  # noqa: E402
from paper_2501_05244_b200 import configs  # noqa: E402

cfg = configs.config(int(os.environ.get("PF_CFG", "4")))
hist = configs.transients(cfg, device=torch.device("cuda"))
k = pf.build_kernel(cfg.lambda_c, cfg.n_bins, cfg.delta_t)
for _ in range(3):
    pf.to_frequency_device(hist, k, cfg.t0)
torch.cuda.synchronize()
ts = []
for _ in range(20):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    pf.to_frequency_device(hist, k, cfg.t0)
    e.record()
    torch.cuda.synchronize()
    ts.append(s.elapsed_time(e))
ms = sorted(ts)[len(ts) // 2]
nbytes = hist.numel() * 4 + k.n_freq * hist.shape[0] * hist.shape[1] * 8
peak = json.load(open("MEASURED_PEAKS.json")) if os.path.exists("MEASURED_PEAKS.json") else {}
print(json.dumps({"cfg": cfg.name, "ms": ms, "min": min(ts), "GBs": nbytes / ms / 1e6, "peaks": peak}))
