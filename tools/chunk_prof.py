"""Per-rank propagation time of an N-GPU shard of config 4 on one GPU: one graph vs the
chunked graphs the overlapped volume gather uses (no collective involved)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_05244_b200 as pf  # noqa: E402
from paper_2501_05244_b200 import configs  # noqa: E402
from paper_2501_05244_b200.pipeline import _Meta  # noqa: E402

cfg = configs.config(4)
k = pf.build_kernel(cfg.lambda_c, cfg.n_bins, cfg.delta_t)
meta = _Meta(k, cfg.relay, cfg.illuminations)
D = cfg.relay.count
rng = np.random.default_rng(0)
coeff = torch.from_numpy(np.exp(2j * np.pi * rng.random((k.n_freq, 1, D))).astype(np.complex64)).cuda()


def timed(fn, reps=7):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    return best


for n in (2, 4, 8):
    planes = 256 // n
    eng = pf.RsdEngine(meta, cfg.grid, plane_range=(0, planes))
    vol = torch.zeros((1, eng.n_voxels), dtype=torch.complex64, device="cuda")
    one = timed(lambda: eng.run_graphed(coeff, vol))
    from paper_2501_05244_b200.distributed import max_chunks
    out = []
    for want in (2, 3, 4):
        c = max_chunks(planes, want, eng.chunk_unit)
        out.append((c, timed(lambda: [eng.run_graphed_chunk(coeff, vol, j, c) for j in range(c)])))
    print(f"N={n} ({planes} planes/rank): one graph {one:.2f} ms; " +
          "; ".join(f"{c} chunks {t:.2f} ms" for c, t in out))
