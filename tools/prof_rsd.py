"""Short rsd run for ncu: config-4 geometry, random slices, n_f frequencies (default 2)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_05244_b200 as pf  # noqa: E402
from paper_2501_05244_b200 import configs  # noqa: E402
from paper_2501_05244_b200.pipeline import _Meta  # noqa: E402

cfg_id = int(os.environ.get("PF_CFG", "4"))
n_f = int(os.environ.get("PF_NF", "2"))
cfg = configs.config(cfg_id)
k = configs.kernel(cfg)
meta = _Meta(k, cfg.relay, cfg.illuminations)
meta.frequencies = meta.frequencies[:n_f]
if cfg.algorithm == "srsd":
    from paper_2501_05244_b200.algorithms import SrsdEngine
    eng = SrsdEngine(meta, cfg.grid)
elif cfg.algorithm == "nursd1":
    from paper_2501_05244_b200.algorithms import Nursd1Engine
    eng = Nursd1Engine(meta, cfg.grid)
else:
    eng = pf.RsdEngine(meta, cfg.grid)
rng = np.random.default_rng(0)
D = cfg.relay.count
coeff = torch.from_numpy(np.exp(2j * np.pi * rng.random((n_f, 1, D))).astype(np.complex64)).cuda()
hist = torch.rand((D, cfg.n_bins), device="cuda")
out = torch.empty((k.n_freq, D), dtype=torch.complex64, device="cuda")
from paper_2501_05244_b200.phasor import TemporalPlan  # noqa: E402
tp = TemporalPlan(k, 0.0, torch.device("cuda"))
for _ in range(2):
    tp.run(hist, out)
    vol = eng.run(coeff)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
vol = eng.run(coeff)
e.record()
torch.cuda.synchronize()
print(f"rsd {n_f} freqs: {s.elapsed_time(e):.3f} ms  ({s.elapsed_time(e)/n_f:.3f} ms/freq)")
