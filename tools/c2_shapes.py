"""Print the config-2 engine's plan shapes (stage-1 3D NUFFT, stage-2 pads / fine grids)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_05244_b200 import configs  # noqa: E402
from paper_2501_05244_b200.pipeline import TransientReconstructor  # noqa: E402

for c in (int(a) for a in (sys.argv[1:] or ["2"])):
    cfg = configs.config(c)
    k = configs.kernel(cfg)
    rec = TransientReconstructor(k, cfg.relay, cfg.illuminations, cfg.grid, t0=cfg.t0,
                                 device=torch.device("cuda"), algorithm=cfg.algorithm,
                                 lattice=getattr(cfg, "lattice", None))
    e = rec.engine
    s1, s2 = e.stage1, e.stage2
    print("config", c, "F", k.n_freq)
    print("stage1 modes", s1.plan.modes3, "fine", s1.plan.mrs, "w", s1.plan.w, "pts", s1.pts.n,
          "px py pz", s1.px, s1.py, getattr(s1, "pz", None))
    ro = getattr(s2, "ro", None) or s2
    print("stage2 px py", s2.px, s2.py, "fine", ro.plan.mrs, "nb", getattr(ro, "nb", None),
          "planes", getattr(ro, "n_planes", None), "count", ro.count)
