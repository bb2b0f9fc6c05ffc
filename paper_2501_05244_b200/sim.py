"""Seeded synthetic transients (input generation for benches and tests; not the hot path).

Semantics follow reference ``sim.simulate`` (sim.py:67-115): each
(illumination p, detector c, scatterer s) return arrives at
``(|x_p - x_s| + |x_s - x_c|)/c``, carries ``albedo/(r1^2 r2^2)`` and is split
linearly over the two bracketing bins.  Differences, documented in DESIGN.md:
returns falling outside the time window are DROPPED instead of raising (the
config-3/4 scenes span more path length than their windows), and
the deposit runs vectorised on the GPU in float32 (the reference takes ~10 h
for config 4 on the CPU).
"""

from __future__ import annotations

import numpy as np
import torch

from .core import SPEED_OF_LIGHT


def simulate_device(scatterers: np.ndarray, albedo: np.ndarray, det_xyz: np.ndarray,
                    ill_xyz: np.ndarray, n_bins: int, delta_t: float, t0: float = 0.0,
                    falloff: bool = True, device=None, chunk: int = 32) -> torch.Tensor:
    """Float32 histograms [n_illum, n_detect, n_bins] on ``device``."""
    device = device or torch.device("cuda")
    det = torch.as_tensor(np.array(det_xyz, dtype=np.float64), device=device)
    ill = torch.as_tensor(ill_xyz, dtype=torch.float64, device=device)
    sc = torch.as_tensor(scatterers, dtype=torch.float64, device=device)
    al = torch.as_tensor(albedo, dtype=torch.float64, device=device)
    n_ill, n_det = ill.shape[0], det.shape[0]
    hist = torch.zeros((n_ill * n_det * n_bins,), dtype=torch.float32, device=device)
    det_off = torch.arange(n_det, device=device, dtype=torch.int64)[:, None] * n_bins
    for p in range(n_ill):
        base = p * n_det * n_bins
        for s0 in range(0, sc.shape[0], chunk):
            s = sc[s0:s0 + chunk]
            r1 = torch.linalg.norm(s - ill[p], dim=1)                       # [S]
            r2 = torch.cdist(det, s)                                        # [D, S]
            amp = al[s0:s0 + chunk][None, :].expand_as(r2)
            if falloff:
                amp = amp / (r1[None, :] ** 2 * r2 ** 2)
            b = ((r1[None, :] + r2) / SPEED_OF_LIGHT - t0) / delta_t
            b0 = torch.floor(b)
            frac = b - b0
            b0 = b0.to(torch.int64)
            ok = (b0 >= 0) & (b0 + 1 <= n_bins - 1)
            idx = (base + det_off + b0).masked_select(ok)
            a = amp.masked_select(ok)
            fr = frac.masked_select(ok)
            hist.index_add_(0, idx, (a * (1.0 - fr)).float())
            hist.index_add_(0, idx + 1, (a * fr).float())
    return hist.view(n_ill, n_det, n_bins)


def add_poisson_noise_device(hist: torch.Tensor, peak_counts: float, seed: int) -> torch.Tensor:
    """Poisson draw of mean ``scale*h`` with ``scale = peak_counts / max(h)`` (sim.py:118-129)."""
    g = torch.Generator(device=hist.device)
    g.manual_seed(int(seed))
    scale = peak_counts / float(hist.max())
    return torch.poisson(hist * scale, generator=g)
