"""One bench step (K1 + reconstruction, graph replay) of BASELINE config $PF_CFG inside a
cudaProfilerStart/Stop range, after warm-up: run under
  ncu --profile-from-start off --metrics gpu__time_duration.sum --csv --log-file X \
      python tools/prof_step.py
to get exactly one step's kernel launches (tools/kernel_roofline.py turns them into
per-kernel roofline rows)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_05244_b200 import configs  # noqa: E402
from paper_2501_05244_b200.pipeline import TransientReconstructor  # noqa: E402

cfg = configs.config(int(os.environ.get("PF_CFG", "4")))
k = configs.kernel(cfg)
dev = torch.device("cuda")
hist = configs.transients(cfg, device=dev)
I, D, T = hist.shape
rec = TransientReconstructor(k, cfg.relay, cfg.illuminations, cfg.grid, t0=cfg.t0, device=dev,
                             algorithm=cfg.algorithm, lattice=getattr(cfg, "lattice", None))


def step():
    rec.temporal.run(hist.view(-1, T), rec.coeff.view(k.n_freq, -1))
    rec.engine.run_graphed(rec.coeff, rec.vol)


for _ in range(3):
    step()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
step()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("step profiled", cfg.name)
