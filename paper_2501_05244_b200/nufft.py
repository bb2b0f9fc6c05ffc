"""Host plans for the GPU NUFFT (geometry only, float64) and the type-1/type-2 drivers.

Same structure as reference ``NufftPlan`` (spectral.py:230-315): a spreading window on a
fine grid ``mr = next_fast_len(max(2m, 2w+2))`` (2x oversampled), the window's transform
divided out of the kept modes, the same ``eps`` contract.  Two windows:

* ``"es"`` (default; BASELINE north star (3)): the exponential of semicircle
  ``exp(beta (sqrt(1 - (d / (w h))^2) - 1))`` with ``beta = 2.30 * 2w`` and
  ``2w = max(6, ceil(log10(1/eps)) + 2)`` taps (8 at the default ``eps = 1e-6``), deconvolved by its
  continuous transform (Gauss-Legendre quadrature).  Measured error against direct sums:
  1e-7 at ``w = 4`` in float64, 3e-7 with float32 weights.
* ``"gaussian"`` (``PF_NUFFT_WINDOW=gaussian``): the reference's own stencil, half-width
  ``w = max(2, ceil(log10(1/eps)) + 2)`` (17 taps at ``eps = 1e-6``),
  ``tau = pi w / (s (s - 1/2) m^2)`` with ``s = mr/m``, and the DISCRETE deconvolution
  ``ker[k] = 1 + 2 sum_j exp(-(j h)^2 / 4 tau) cos(k j h)`` (points on fine-grid nodes exact).

Both use the per-point stencil anchors ``i0`` (nearest fine node) and centre-tap offsets
``d0`` of spectral.py:281-303 and taps ``-w..w``; the tile buckets of the gather-spread
kernel are computed here once per geometry.
"""

from __future__ import annotations

import ctypes
import math
import os

import numpy as np
import torch

from . import _device as dev
from . import _lib
from ._fastlen import next_fast_len
from .core import _require

_EPS_MIN, _EPS_MAX = 1e-14, 1e-1
_COORD_TOL = 1e-9
TILE_2D = (1, 16, 16)
TILE_3D = (4, 8, 8)
_T2_FUSED = os.environ.get("PF_T2_FUSED", "1") != "0"
_T1_SKIP_ZERO = os.environ.get("PF_T1_SKIP_ZERO", "1") != "0"
DEFAULT_WINDOW = os.environ.get("PF_NUFFT_WINDOW", "es")
_ES_BETA_PER_TAP = 2.30


def es_half_width(eps: float) -> int:
    """Half-width w of the exponential-of-semicircle window: 2w = ceil(log10(1/eps)) + 2 taps,
    at least 6 (1e-5 against direct sums), so that even the loosest request stays inside the
    1e-4 parity gate against the reference, whose Gaussian over-delivers at loose eps."""
    return max(3, -(-(math.ceil(math.log10(1.0 / eps)) + 2) // 2))


def es_transform(w: int, xi: np.ndarray) -> np.ndarray:
    """Continuous transform of exp(beta (sqrt(1 - (x/w)^2) - 1)) on |x| <= w (grid units) at
    the angular frequencies ``xi`` (radians per cell): 64-node Gauss-Legendre, float64."""
    xg, wg = np.polynomial.legendre.leggauss(64)
    x = xg * w
    phi = np.exp(_ES_BETA_PER_TAP * 2 * w * (np.sqrt(1.0 - xg * xg) - 1.0)) * wg * w
    return (phi[None, :] * np.cos(np.outer(xi, x))).sum(axis=1)


class NufftPlan:
    """Plan for modes ``(m_y, m_x)`` or ``(m_z, m_y, m_x)`` at accuracy ``eps``."""

    def __init__(self, modes, eps: float, device, window: str | None = None):
        modes = tuple(int(m) for m in modes)
        _require(len(modes) in (2, 3), "supported dimensionalities are 2 and 3")
        _require(all(m >= 1 for m in modes), "mode counts must be >= 1")
        _require(math.isfinite(eps) and _EPS_MIN <= eps <= _EPS_MAX,
                 f"accuracy target must lie in [{_EPS_MIN:g}, {_EPS_MAX:g}]")
        self.window = DEFAULT_WINDOW if window is None else window
        _require(self.window in ("es", "gaussian"), "window must be 'es' or 'gaussian'")
        self.dim = len(modes)
        self.modes3 = (1,) * (3 - self.dim) + modes
        if self.window == "es":
            self.w = es_half_width(eps)
        else:
            self.w = max(2, math.ceil(math.log10(1.0 / eps)) + 2)
        _require(self.w <= 16, "accuracy target too tight for the GPU stencil (w <= 16)")
        self.device = device
        mrs, taus, kers = [], [], []
        for m in self.modes3:
            if m == 1 and len(mrs) < 3 - self.dim:
                mrs.append(1)
                taus.append(1.0)
                kers.append(np.ones(1))
                continue
            mr = next_fast_len(max(2 * m, 2 * self.w + 2))
            s = mr / m
            tau = math.pi * self.w / (s * (s - 0.5) * m * m)
            h = 2.0 * math.pi / mr
            k = np.arange(m) - m // 2
            if self.window == "es":
                ker = es_transform(self.w, k * h)
            else:
                j = np.arange(1, self.w + 1)
                ker = 1.0 + 2.0 * (np.exp(-(j * h) ** 2 / (4.0 * tau))[None, :]
                                   * np.cos(np.outer(k, j * h))).sum(axis=1)
            assert (ker > 0).all()
            mrs.append(mr)
            taus.append(tau)
            kers.append(ker)
        self.mrs = tuple(mrs)
        self.taus = tuple(taus)
        self.tile = TILE_2D if self.dim == 2 else TILE_3D
        g = _lib.PfNufftGeom()
        g.dim, g.w = self.dim, self.w
        g.window = 1 if self.window == "es" else 0
        g.beta = _ES_BETA_PER_TAP * 2 * self.w
        for a in range(3):
            g.mr[a] = self.mrs[a]
            g.m[a] = self.modes3[a]
            g.h[a] = 2.0 * math.pi / self.mrs[a]
            g.inv4tau[a] = 1.0 / (4.0 * self.taus[a])
            g.inv_hw[a] = 1.0 / (self.w * g.h[a])
            g.tile[a] = self.tile[a]
            g.ntiles[a] = -(-self.mrs[a] // self.tile[a])
        self.geom = g
        self.kers = [torch.from_numpy(k.astype(np.float32)).to(device) for k in kers]
        self.fine_elems = int(np.prod(self.mrs))
        self.mode_elems = int(np.prod(self.modes3))
        # type-1 finish on the register path: square 2D modes m in 128..1024, mr = 2m
        m2 = self.modes3[2]
        self.pow2_finish = (self.dim == 2 and self.modes3[1] == m2 and m2 in (128, 256, 512, 1024)
                            and self.mrs[1] == 2 * m2 and self.mrs[2] == 2 * m2
                            and os.environ.get("PF_NUFFT_FAST", "1") != "0")
        self._rt = None
        # natural fine-grid slots of the centred modes per transformed axis
        self.kept = [dev.kept_ranges(m, mr) for m, mr in
                     zip(self.modes3[3 - self.dim:], self.mrs[3 - self.dim:])]

    @property
    def gref(self):
        return ctypes.byref(self.geom)

    # -- per-geometry point data ------------------------------------------------------
    def points(self, pts: np.ndarray, cell_sorted: bool = False) -> "NufftPoints":
        return NufftPoints(self, pts, cell_sorted)


def check_points(pts, d: int) -> np.ndarray:
    """Torus coordinates [L, d] in [-pi, pi) (reference spectral.py:318-329)."""
    pts = np.asarray(pts, dtype=np.float64)
    if pts.ndim == 1:
        pts = pts[:, None]
    _require(pts.ndim == 2 and pts.shape[1] == d, f"points must be [L, {d}] for {d}-dimensional modes")
    _require(pts.shape[0] >= 1, "need at least one point")
    _require(bool(np.isfinite(pts).all()), "point coordinates must be finite")
    _require(bool((pts >= -math.pi - _COORD_TOL).all() and (pts < math.pi + _COORD_TOL).all()),
             "point coordinates must lie in [-pi, pi)")
    return pts


class NufftPoints:
    """Stencil anchors + tile buckets of one point set under one plan (device tensors).

    ``cell_sorted=True`` (type-2 readouts) stores the points ordered by their stencil
    anchor so neighbouring threads gather overlapping fine-grid patches; ``perm`` maps
    the stored order back to the caller's point index.
    """

    def __init__(self, plan: NufftPlan, pts: np.ndarray, cell_sorted: bool = False):
        pts = check_points(pts, plan.dim)
        L = pts.shape[0]
        self.n = L
        self.order = None
        i0 = np.zeros((L, 3), dtype=np.int64)
        d0 = np.zeros((L, 3), dtype=np.float64)
        for a in range(3 - plan.dim, 3):
            # mode axis a (z, y, x order) pairs with point column (2 - a) (x is column 0)
            x = pts[:, 2 - a]
            mr = plan.mrs[a]
            h = 2.0 * math.pi / mr
            xi = x - 2.0 * math.pi * np.floor(x / (2.0 * math.pi))
            k = np.floor(xi / h + 0.5).astype(np.int64)
            i0[:, a] = k
            d0[:, a] = k * h - xi
        dv = plan.device
        self.perm = None
        if cell_sorted:
            order = np.lexsort([i0[:, 2], i0[:, 1], i0[:, 0]])
            i0, d0 = i0[order], d0[order]
            self.order = order
            self.perm = torch.from_numpy(order.astype(np.int32)).to(dv)
        self.i0 = torch.from_numpy(i0.astype(np.int32)).to(dv)
        self.d0 = torch.from_numpy(d0.astype(np.float32)).to(dv)
        self._i0_host = i0
        self.plan = plan
        self._tiles = None

    def touched_runs(self):
        """Per transformed axis: runs (start, length) of the fine slots some stencil of these
        points touches -- the shortest covering arc of the torus, split at the seam.  Every
        other slot of a spread fine grid is zero."""
        if getattr(self, "_runs", None) is None:
            p = self.plan
            runs = []
            for a in range(3 - p.dim, 3):
                mr, w = p.mrs[a], p.w
                touched = np.zeros(mr, dtype=bool)
                i0 = np.unique(self._i0_host[:, a] % mr)
                for j in range(-w, w + 1):
                    touched[(i0 + j) % mr] = True
                if touched.all():
                    runs.append([(0, mr)])
                    continue
                idx = np.flatnonzero(touched)
                gaps = np.diff(np.append(idx, idx[0] + mr)) - 1
                g = int(np.argmax(gaps))
                start, n = int(idx[(g + 1) % idx.size]), mr - int(gaps[g])
                runs.append([(start, n)] if start + n <= mr else
                            [(0, start + n - mr), (start, mr - start)])
            self._runs = runs
        return self._runs

    def tiles(self):
        """CSR (tile_start, tile_pts) of the tiles each point's stencil touches."""
        if self._tiles is not None:
            return self._tiles
        p = self.plan
        w = p.w
        per_axis = []
        for a in range(3):
            if p.mrs[a] == 1:
                per_axis.append(np.zeros((self.n, 1), dtype=np.int64))
                continue
            cells = (self._i0_host[:, a][:, None] + np.arange(-w, w + 1)[None, :]) % p.mrs[a]
            t = np.sort(cells // p.tile[a], axis=1)
            dup = np.zeros_like(t, dtype=bool)
            dup[:, 1:] = t[:, 1:] == t[:, :-1]
            t[dup] = -1
            keep = (~dup).sum(axis=1).max()
            t = -np.sort(-t, axis=1)[:, :keep]   # valid ids first, -1 padding last
            per_axis.append(t)
        nt = [int(p.geom.ntiles[a]) for a in range(3)]
        tz, ty, tx = per_axis
        comb = (tz[:, :, None, None] * nt[1] + ty[:, None, :, None]) * nt[2] + tx[:, None, None, :]
        valid = (tz[:, :, None, None] >= 0) & (ty[:, None, :, None] >= 0) & (tx[:, None, None, :] >= 0)
        comb = np.where(valid, comb, -1).reshape(self.n, -1)
        pid = np.broadcast_to(np.arange(self.n)[:, None], comb.shape)
        sel = comb >= 0
        tid, pts = comb[sel], pid[sel]
        order = np.argsort(tid, kind="stable")
        tid, pts = tid[order], pts[order]
        ntot = nt[0] * nt[1] * nt[2]
        start = np.zeros(ntot + 1, dtype=np.int64)
        np.cumsum(np.bincount(tid, minlength=ntot), out=start[1:])
        dv = p.device
        self._tiles = (torch.from_numpy(start.astype(np.int32)).to(dv),
                       torch.from_numpy(pts.astype(np.int32)).to(dv))
        return self._tiles


def type1(plan: NufftPlan, pts: NufftPoints, vals: torch.Tensor, nv: int, val_stride: int,
          out: torch.Tensor, out_stride: int, fine: torch.Tensor | None = None,
          transpose: bool = False, stream=None) -> torch.Tensor:
    """U[v][k] = sum_l vals[v][l] exp(-1j k.x_l) for centred k (spectral.py:336-358).

    ``out`` receives natural-order modes ([v][..modes..], or [v][x][y] with
    ``transpose`` in 2D).  ``fine`` is scratch [nv][prod(mr)] complex64.
    """
    if fine is None:
        fine = torch.empty((nv, plan.fine_elems), dtype=torch.complex64, device=plan.device)
    ts, tp = pts.tiles()
    s = dev.stream_ptr(stream)
    _lib.call("pf_nufft_spread", plan.gref, dev.ptr(pts.i0), dev.ptr(pts.d0), dev.ptr(ts),
              dev.ptr(tp), dev.ptr(vals), val_stride, nv, dev.ptr(fine), plan.fine_elems, s)
    kz, ky, kx = plan.kers
    if transpose and plan.pow2_finish:
        # register path: split fine-grid FFT that forms only the kept modes, fused
        # with the deconvolution (pf_nufft_type1_finish_pow2)
        m = plan.modes3[2]
        need = nv * m * 2 * m
        if plan._rt is None or plan._rt.numel() < need:
            plan._rt = torch.empty((need,), dtype=torch.complex64, device=plan.device)
        _lib.call("pf_nufft_type1_finish_pow2", plan.gref, dev.ptr(fine), plan.fine_elems, nv,
                  dev.ptr(plan._rt), dev.fft_plan(2 * m, plan.device).ref,
                  dev.fft_plan(m, plan.device).ref, dev.ptr(ky), dev.ptr(kx), dev.ptr(out),
                  out_stride, s)
        return out
    shape = plan.mrs[3 - plan.dim:]
    # only the kept modes are gathered: transform only the lines that reach them
    # ... and, before an axis is transformed, only along lines through cells the spreading
    # touched (the rest of the grid is zero and stays zero)
    dev.fftn_pruned(fine, shape, nv, -1, plan.kept, True, stream,
                    pts.touched_runs() if _T1_SKIP_ZERO else None)
    _lib.call("pf_nufft_deconv", plan.gref, dev.ptr(fine), plan.fine_elems, dev.ptr(kz),
              dev.ptr(ky), dev.ptr(kx), nv, dev.ptr(out), out_stride, int(transpose), s)
    return out


def stencil_window(plan: NufftPlan, point_sets) -> tuple[int, int, int, int]:
    """(col0, ncols, row0, nrows): per axis the shortest arc of the fine-grid torus that holds
    every stencil cell (anchor - w .. anchor + w) of every point in ``point_sets``
    (NufftPoints of a 2D plan) -- all a type-2 readout of these points ever reads."""
    out = []
    for a in (2, 1):
        mr, w = plan.mrs[a], plan.w
        touched = np.zeros(mr, dtype=bool)
        for ps in point_sets:
            i0 = np.unique(ps._i0_host[:, a] % mr)
            for j in range(-w, w + 1):
                touched[(i0 + j) % mr] = True
        if touched.all() or not touched.any():
            out += [0, mr]
            continue
        # longest circular run of untouched cells; the window is its complement
        idx = np.flatnonzero(touched)
        gaps = np.diff(np.append(idx, idx[0] + mr)) - 1
        g = int(np.argmax(gaps))
        start = int(idx[(g + 1) % idx.size])
        out += [start, mr - int(gaps[g])]
    return tuple(out)


def place_and_inverse(plan: NufftPlan, S: torch.Tensor, nv: int, s_stride: int,
                      fine: torch.Tensor, stream=None, window=None) -> torch.Tensor:
    """Type-2 first half (spectral.py:373-375): fine = ifftn(place(S / ker)) * prod(mr).
    ``window`` (``stencil_window``): the caller reads only these fine cells, the others may
    be left unformed."""
    kz, ky, kx = plan.kers
    if plan.dim == 2 and _T2_FUSED:
        # place + pruned inverse FFT in two fused passes
        c0, nc, r0, nr = window if window is not None else (0, plan.mrs[2], 0, plan.mrs[1])
        _lib.call("pf_nufft_type2_start_2d_win", plan.gref, dev.ptr(S), s_stride, dev.ptr(ky),
                  dev.ptr(kx), nv, dev.ptr(fine), plan.fine_elems,
                  dev.fft_plan(plan.mrs[2], plan.device).ref,
                  dev.fft_plan(plan.mrs[1], plan.device).ref, c0, nc, r0, nr,
                  dev.stream_ptr(stream))
        return fine
    _lib.call("pf_nufft_place", plan.gref, dev.ptr(S), s_stride, dev.ptr(kz), dev.ptr(ky),
              dev.ptr(kx), nv, dev.ptr(fine), plan.fine_elems, 0, dev.stream_ptr(stream))
    shape = plan.mrs[3 - plan.dim:]
    # the placed grid is zero off the mode slots: skip the lines that are all zero
    dev.fftn_pruned(fine, shape, nv, +1, plan.kept, False, stream)
    return fine
