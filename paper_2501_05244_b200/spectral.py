"""GPU drop-ins for the reference transform primitives (reference ``spectral.py``).

``cfft_n`` / ``cifft_n`` / ``cfft_2d`` / ``cifft_2d`` (:107-124), ``sfft_1d`` /
``sfft_2d`` / ``sfft_2d_centered`` (:183-218), ``nufft1`` / ``nufft2`` (:336-381)
with the reference signatures; numpy in, numpy out (complex128), computed in
complex64 on the GPU by the same kernels the reconstructions use.  ``next_fast_len``
is re-exported as the reference does.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _device as dev
from . import _lib
from . import nufft as nu
from ._fastlen import next_fast_len
from .core import _require

__all__ = ["cfft_n", "cifft_n", "cfft_2d", "cifft_2d", "sfft_1d", "sfft_2d", "sfft_2d_centered",
           "nufft1", "nufft2", "next_fast_len", "fft_2d", "ifft_2d", "dft_2d", "idft_2d"]


def _to_dev(a) -> torch.Tensor:
    device = dev.require_cuda()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.complex64)).to(device)


def _centered(u, axes, direction):
    u = np.asarray(u, dtype=np.complex128)
    axes = tuple(sorted(a % u.ndim for a in axes))
    _require(len(axes) <= 3, "at most three transform axes")
    moved = np.moveaxis(u, axes, tuple(range(u.ndim - len(axes), u.ndim)))
    shape = moved.shape[u.ndim - len(axes):]
    nb = int(np.prod(moved.shape[:u.ndim - len(axes)])) if u.ndim > len(axes) else 1
    n = (1,) * (3 - len(shape)) + tuple(shape)
    x = _to_dev(moved)
    y = torch.empty_like(x)
    s = dev.stream_ptr()
    # ifftshift (centred -> natural), FFT, fftshift (natural -> centred)
    _lib.call("pf_roll", dev.ptr(x), dev.ptr(y), nb, *n, *(m // 2 for m in n), s)
    total = int(np.prod(shape))
    dev.fftn_natural(y, tuple(shape), nb, direction, (1.0 / total) if direction > 0 else 1.0)
    _lib.call("pf_roll", dev.ptr(y), dev.ptr(x), nb, *n, *(m - m // 2 for m in n), s)
    out = x.cpu().numpy().astype(np.complex128).reshape(moved.shape)
    return np.moveaxis(out, tuple(range(u.ndim - len(axes), u.ndim)), axes)


def cfft_n(u, axes):
    """Centred-index forward DFT over ``axes`` (reference spectral.py:107-109)."""
    return _centered(u, axes, -1)


def cifft_n(u, axes):
    """Centred-index inverse DFT over ``axes`` with 1/N (reference spectral.py:112-114)."""
    return _centered(u, axes, +1)


def fft_2d(u):
    """Forward 2D DFT over the last two axes, natural order, unnormalised (spectral.py:97-99)."""
    u = np.asarray(u, dtype=np.complex128)
    _require(u.ndim >= 2, "fft_2d takes an array with at least two axes")
    x = _to_dev(u)
    dev.fft2_natural(x.view(-1), u.shape[-2], u.shape[-1], int(np.prod(u.shape[:-2])), -1)
    return x.cpu().numpy().astype(np.complex128)


def ifft_2d(u):
    """Inverse of :func:`fft_2d` with 1/(ny nx) (spectral.py:102-104)."""
    u = np.asarray(u, dtype=np.complex128)
    _require(u.ndim >= 2, "ifft_2d takes an array with at least two axes")
    x = _to_dev(u)
    ny, nx = u.shape[-2], u.shape[-1]
    dev.fft2_natural(x.view(-1), ny, nx, int(np.prod(u.shape[:-2])), +1, 1.0 / (ny * nx))
    return x.cpu().numpy().astype(np.complex128)


def dft_2d(u):
    """2D DFT (spectral.py:77-84; the reference forms it by explicit matrices, same values)."""
    u = np.asarray(u)
    _require(u.ndim == 2, "dft_2d takes a 2D array")
    return fft_2d(u)


def idft_2d(u):
    """Inverse of :func:`dft_2d` scaled by 1/(ny nx) (spectral.py:87-94)."""
    u = np.asarray(u)
    _require(u.ndim == 2, "idft_2d takes a 2D array")
    return ifft_2d(u)


def cfft_2d(u):
    return cfft_n(u, axes=(-2, -1))


def cifft_2d(u):
    return cifft_n(u, axes=(-2, -1))


def sfft_1d(u, alpha: float, offset: int = 0, axis: int = -1):
    """``U[k] = sum_n u[n] exp(-2j pi alpha (n-o)(k-o)/M)`` (reference spectral.py:183-193)."""
    import math
    from .algorithms import _sfft_tables
    u = np.asarray(u, dtype=np.complex128)
    moved = np.moveaxis(u, axis, -1)
    m = moved.shape[-1]
    _require(m >= 1, "transform length must be >= 1")
    _require(math.isfinite(alpha) and alpha != 0.0, "scale factor must be finite and nonzero")
    _require(0 <= offset < m, "index offset must lie in [0, length)")
    q = next_fast_len(max(1, 2 * m - 1))
    chirp, khat = _sfft_tables(m, alpha, offset, q)
    device = dev.require_cuda()
    nl = int(np.prod(moved.shape[:-1])) if moved.ndim > 1 else 1
    x = _to_dev(moved.reshape(nl, m))
    y = torch.empty_like(x)
    ch = torch.from_numpy(chirp).to(device)
    kh = torch.from_numpy(khat).to(device)
    plan = dev.fft_plan(q, device)
    _lib.call("pf_bluestein_lines", dev.ptr(x), 0, m, 1, m, 0, dev.ptr(y), 0, m, 1, 0, m, nl, 1,
              plan.ref, dev.ptr(ch), dev.ptr(kh), dev.stream_ptr())
    out = y.cpu().numpy().astype(np.complex128).reshape(moved.shape)
    return np.moveaxis(out, -1, axis)


def sfft_2d(u, alpha: float, beta: float | None = None, offsets=(0, 0)):
    """x pass (alpha, offsets[1]) then y pass (beta, offsets[0]) (reference spectral.py:196-206)."""
    beta = alpha if beta is None else beta
    return sfft_1d(sfft_1d(u, alpha, offsets[1], -1), beta, offsets[0], -2)


def sfft_2d_centered(u, alpha: float, beta: float | None = None):
    ny, nx = np.asarray(u).shape[-2:]
    return sfft_2d(u, alpha, beta, offsets=(ny // 2, nx // 2))


def nufft1(points, values, modes, eps: float):
    """Type 1, exponent -1j, points -> centred modes (reference spectral.py:336-358)."""
    modes = tuple(int(m) for m in modes)
    _require(1 <= len(modes) <= 3, "supported dimensionalities are 1, 2, 3")
    d = len(modes)
    pts = nu.check_points(points, d)
    vals = np.asarray(values, dtype=np.complex128)
    _require(vals.shape == (pts.shape[0],), "values must be [L] matching the points")
    _require(bool(np.isfinite(vals).all()), "values must be finite")
    m2 = modes if d > 1 else (1,) + modes
    p2 = pts if d > 1 else np.column_stack([pts[:, 0], np.zeros(pts.shape[0])])
    device = dev.require_cuda()
    plan = nu.NufftPlan(m2, eps, device)
    out = torch.empty((plan.mode_elems,), dtype=torch.complex64, device=device)
    nu.type1(plan, plan.points(p2), _to_dev(vals), 1, vals.size, out, plan.mode_elems)
    nat = out.cpu().numpy().astype(np.complex128).reshape(m2)
    return np.fft.fftshift(nat).reshape(modes)   # natural -> centred slots


def nufft2(coefficients, points, eps: float):
    """Type 2, exponent +1j, centred modes -> points (reference spectral.py:361-381); 1D-3D."""
    coeff = np.asarray(coefficients, dtype=np.complex128)
    _require(1 <= coeff.ndim <= 3, "mode array must be 1D, 2D, or 3D")
    _require(bool(np.isfinite(coeff).all()), "coefficients must be finite")
    pts = nu.check_points(points, coeff.ndim)
    if coeff.ndim == 1:   # 1D as a single-row 2D problem (as nufft1)
        coeff = coeff[None, :]
        pts = np.column_stack([pts[:, 0], np.zeros(pts.shape[0])])   # x pairs with the last axis
    device = dev.require_cuda()
    plan = nu.NufftPlan(coeff.shape, eps, device)
    S = _to_dev(np.fft.ifftshift(coeff))         # centred slots -> natural order
    fine = torch.empty((1, plan.fine_elems), dtype=torch.complex64, device=device)
    nu.place_and_inverse(plan, S, 1, plan.mode_elems, fine)
    P = plan.points(pts)
    out = torch.zeros((pts.shape[0],), dtype=torch.complex64, device=device)
    _lib.call("pf_nufft_interp", plan.gref, dev.ptr(P.i0), dev.ptr(P.d0), pts.shape[0],
              dev.ptr(fine), dev.ptr(out), dev.stream_ptr())
    return out.cpu().numpy().astype(np.complex128)
