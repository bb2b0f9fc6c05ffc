"""K1 timing at config 1 (T = 2048, 4096 traces) with and without a preceding L2 flush."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_05244_b200 as pf  # noqa
from paper_2501_05244_b200 import configs  # noqa
from paper_2501_05244_b200.phasor import TemporalPlan  # noqa
cfg = configs.config(int(os.environ.get("PF_CFG", "1")))
k = configs.kernel(cfg)
h = configs.transients(cfg, device=torch.device("cuda"))
I, D, T = h.shape
tp = TemporalPlan(k, cfg.t0, torch.device("cuda"))
out = torch.empty((k.n_freq, D), dtype=torch.complex64, device="cuda")
flush = torch.empty(4 * torch.cuda.get_device_properties(0).L2_cache_size // 4, device="cuda")
for fl in (False, True, False, True):
    ts = []
    for _ in range(10):
        if fl:
            flush.fill_(1.0)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); tp.run(h.view(-1, T), out); e.record(); torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    print("flush" if fl else "warm ", ["%.3f" % t for t in ts])
