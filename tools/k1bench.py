"""K1 variants on the config-4 capture: device time and HBM fraction (env PF_K1_* select)."""
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
ref = pf.to_frequency_device(hist, k, cfg.t0)
torch.cuda.synchronize()
res = {}
for name, env in [("tma_g4_s2", {"PF_K1_TMA": "1", "PF_K1_G": "4", "PF_K1_S": "2"}),
                  ("tma_g2_s3", {"PF_K1_TMA": "1", "PF_K1_G": "2", "PF_K1_S": "3"}),
                  ("tma_g2_s2", {"PF_K1_TMA": "1", "PF_K1_G": "2", "PF_K1_S": "2"}),
                  ("tma_g1_s4", {"PF_K1_TMA": "1", "PF_K1_G": "1", "PF_K1_S": "4"}),
                  ("ldg", {})]:
    for key in ("PF_K1_G", "PF_K1_S", "PF_K1_TMA"):
        os.environ.pop(key, None)
    os.environ.update(env)
    out = pf.to_frequency_device(hist, k, cfg.t0)
    torch.cuda.synchronize()
    err = float((out - ref).abs().max() / ref.abs().max())
    ts = []
    for _ in range(10):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        pf.to_frequency_device(hist, k, cfg.t0)
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ms = sorted(ts)[len(ts) // 2]
    nbytes = hist.numel() * 4 + k.n_freq * hist.shape[0] * hist.shape[1] * 8
    res[name] = {"ms": ms, "GBs": nbytes / ms / 1e6, "frac": nbytes / ms / 1e6 / 6456.5,
                 "max_rel_dev_vs_default": err}
print(json.dumps(res, indent=1))
