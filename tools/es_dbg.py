import os, sys, math
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_05244_b200 import nufft as nu, _lib, _device as dev
rng = np.random.default_rng(1)
d = torch.device("cuda")
for wdw in ("es", "gaussian"):
    modes, eps = (20, 24), 1e-6
    plan = nu.NufftPlan(modes, eps, d, window=wdw)
    L = 50
    pts = rng.uniform(-np.pi, np.pi, size=(L, 2))
    vals = (rng.normal(size=L) + 1j * rng.normal(size=L)).astype(np.complex64)
    P = plan.points(pts)
    ts, tp = P.tiles()
    fine = torch.full((1, plan.fine_elems), complex(np.nan, np.nan), dtype=torch.complex64, device=d)
    v = torch.from_numpy(vals).to(d)
    _lib.call("pf_nufft_spread", plan.gref, dev.ptr(P.i0), dev.ptr(P.d0), dev.ptr(ts), dev.ptr(tp),
              dev.ptr(v), L, 1, dev.ptr(fine), plan.fine_elems, 0)
    torch.cuda.synchronize()
    got = fine.cpu().numpy().reshape(plan.mrs[1], plan.mrs[2])
    # numpy spread
    w = plan.w
    ref = np.zeros((plan.mrs[1], plan.mrs[2]), complex)
    def win(a, dl):
        if wdw == "gaussian":
            return np.exp(-dl * dl / (4 * plan.taus[a]))
        h = 2 * np.pi / plan.mrs[a]
        z = dl / (w * h); q = 1 - z * z
        return np.where(q > 0, np.exp(2.3 * 2 * w * (np.sqrt(np.maximum(q, 0)) - 1)), 0.0)
    i0 = P._i0_host
    offs = np.arange(-w, w + 1)
    for l in range(L):
        wy = win(1, (i0[l, 1] + offs) * (2 * np.pi / plan.mrs[1]) - (pts[l, 1] % (2 * np.pi)))
        wx = win(2, (i0[l, 2] + offs) * (2 * np.pi / plan.mrs[2]) - (pts[l, 0] % (2 * np.pi)))
        ref[np.ix_((i0[l, 1] + offs) % plan.mrs[1], (i0[l, 2] + offs) % plan.mrs[2])] += vals[l] * np.outer(wy, wx)
    print(wdw, "w", w, "mrs", plan.mrs, "spread relerr", np.linalg.norm(got - ref) / np.linalg.norm(ref),
          "nan", np.isnan(got).sum(), "sum ratio", np.abs(got).sum() / np.abs(ref).sum())
    print(" geom", plan.geom.window, plan.geom.beta, list(plan.geom.inv_hw), list(plan.geom.h), plan.geom.w)
