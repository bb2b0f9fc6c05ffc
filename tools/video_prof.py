import os, sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2501_05244_b200 as pf
from paper_2501_05244_b200 import configs
from paper_2501_05244_b200.pipeline import _Meta
cfg = configs.config(4)
k = pf.build_kernel(cfg.lambda_c, cfg.n_bins, cfg.delta_t)
meta = _Meta(k, cfg.relay, cfg.illuminations)
nf = 8
meta.frequencies = meta.frequencies[:nf]
D = cfg.relay.count
rng = np.random.default_rng(0)
coeff = torch.from_numpy(np.exp(2j*np.pi*rng.random((nf, 1, D))).astype(np.complex64)).cuda()
for times in (None, np.array([0.0, 1e-10]), np.array([0.0, 1e-10, 2e-10, 3e-10])):
    eng = pf.RsdEngine(meta, cfg.grid, times=times)
    for _ in range(2): eng.run(coeff)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); eng.run(coeff); e.record(); torch.cuda.synchronize()
    print("frames", 1 if times is None else times.size, f"{s.elapsed_time(e):.2f} ms for {nf} freqs")
