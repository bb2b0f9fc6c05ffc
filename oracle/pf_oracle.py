"""CPU oracle for the phasor-field reconstruction hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package imports this
module; it is used by ``tests/`` (parity checker), ``__graft_entry__.smoke()``
(checker) and ``bench.py`` (the ``cpu_baseline`` leg and ``--impl reference``).

It is a float64 numpy restatement of the reference algorithms in
``/root/reference/pkg/src/phasorfield`` (the reference is pure Python and
cannot travel to the GPU box).  Every function cites the reference lines it
follows.  Structure differs from the reference (depth planes are batched
through numpy's FFT, the NUFFT spreads with ``np.add.at`` instead of a
per-point loop) but sizes, index conventions and the order of frequency /
illumination accumulation are the reference's.

Pinning: ``tests/test_oracle_golden.py`` checks this module against golden
vectors produced by running the reference itself in the build container
(``tests/golden/make_golden.py``), plus the reference's own known-answer tests
(``test_phasor.py:29-30,94-115``, ``test_spectral.py:77-186``,
``test_reconstruct.py:103-113``).

Inputs are duck-typed: any object exposing the reference's field names
(``frequencies``, ``coefficients``, ``relay.kind`` ...) works, so both the
reference's containers and the engine's mirror types can be fed in.
Functions return plain numpy arrays (the ``field`` of the reference's
``ReconstructionVolume``).
"""

from __future__ import annotations

import math
from functools import reduce

import numpy as np
from scipy.fft import next_fast_len

C = 299792458.0      # reference core.py:28
SIGN = +1.0          # reference core.py:35 (PROPAGATION_SIGN)


class OracleError(ValueError):
    pass


def _need(ok, msg):
    if not ok:
        raise OracleError(msg)


# ---------------------------------------------------------------------------
# phasor kernel and temporal transform (reference phasor.py:72-127)
# ---------------------------------------------------------------------------


def build_kernel(lambda_c, n_bins, delta_t, threshold=0.01):
    """Bins, angular frequencies and Gaussian weights (phasor.py:84-89)."""
    omega_c = 2.0 * math.pi * C / lambda_c
    sigma = C / (5.0 * lambda_c)
    b = np.arange(1, n_bins // 2 + 1)
    om = 2.0 * math.pi * b / (n_bins * delta_t)
    wt = np.exp(-((om - omega_c) ** 2) / (2.0 * sigma * sigma))
    keep = wt >= threshold
    _need(keep.any(), "no DFT bin reaches the retention threshold")
    return b[keep], om[keep], wt[keep]


def to_frequency(hist, bins, freqs, weights, t0):
    """``FFT(h)[bins] * w * exp(-1j w t0)`` over the last axis (phasor.py:119-121)."""
    spec = np.fft.fft(np.asarray(hist, dtype=np.float64), axis=-1)
    return spec[..., bins] * weights * np.exp(-1j * freqs * t0)


def to_frequency_direct(hist, bins, freqs, weights, t0, delta_t):
    """Direct weighted DFT, the reference test oracle (test_phasor.py:105-115)."""
    h = np.asarray(hist, dtype=np.float64)
    t = t0 + np.arange(h.shape[-1]) * delta_t
    return np.einsum("...b,fb->...f", h, np.exp(-1j * np.outer(freqs, t))) * weights


# ---------------------------------------------------------------------------
# centred FFTs, scaled FFT, NUFFT (reference spectral.py:107-381)
# ---------------------------------------------------------------------------


def cfft(u, axes):
    """Centred-index DFT (spectral.py:107-109)."""
    return np.fft.fftshift(np.fft.fftn(np.fft.ifftshift(u, axes=axes), axes=axes), axes=axes)


def cifft(u, axes):
    """Centred-index inverse DFT with 1/N (spectral.py:112-114)."""
    return np.fft.fftshift(np.fft.ifftn(np.fft.ifftshift(u, axes=axes), axes=axes), axes=axes)


def cfft2(u):
    return cfft(u, (-2, -1))


def cifft2(u):
    return cifft(u, (-2, -1))


def sfft_tables(m, alpha, offset):
    """Chirp and embedded-kernel spectrum of one scaled DFT (spectral.py:143-158)."""
    n = np.arange(m, dtype=np.float64) - offset
    chirp = np.exp(-1j * np.pi * alpha * n * n / m)
    q = next_fast_len(max(1, 2 * m - 1))
    lags = np.arange(1 - m, m)
    kern = np.zeros(q, dtype=np.complex128)
    kern[lags % q] = np.exp(1j * np.pi * alpha * lags * lags / m)
    return chirp, np.fft.fft(kern), q


def sfft_1d(u, alpha, offset=0, axis=-1):
    """``U[k] = sum_n u[n] exp(-2j pi alpha (n-o)(k-o)/M)`` (spectral.py:160-168,183-193)."""
    u = np.moveaxis(np.asarray(u, dtype=np.complex128), axis, -1)
    m = u.shape[-1]
    chirp, kfft, q = sfft_tables(m, alpha, offset)
    buf = np.zeros(u.shape[:-1] + (q,), dtype=np.complex128)
    buf[..., :m] = u * chirp
    conv = np.fft.ifft(np.fft.fft(buf, axis=-1) * kfft, axis=-1)
    return np.moveaxis(conv[..., :m] * chirp, -1, axis)


def sfft_2d_centered(u, alpha, beta=None):
    """x pass then y pass with offsets M//2 (spectral.py:196-218)."""
    beta = alpha if beta is None else beta
    ny, nx = np.shape(u)[-2:]
    return sfft_1d(sfft_1d(u, alpha, nx // 2, -1), beta, ny // 2, -2)


def scaled_dft(u, alpha, offset=0):
    """Quadratic-time scaled DFT (reference oracle.py:31-38)."""
    u = np.asarray(u, dtype=np.complex128)
    n = np.arange(u.size) - offset
    return np.exp(-2j * np.pi * alpha * np.outer(n, n) / u.size) @ u


class NufftPlan:
    """Gaussian-gridding geometry for one (modes, eps) pair (spectral.py:249-303)."""

    def __init__(self, modes, eps):
        _need(1 <= len(modes) <= 3, "supported dimensionalities are 1, 2, 3")
        _need(math.isfinite(eps) and 1e-14 <= eps <= 1e-1, "accuracy target out of range")
        self.modes = tuple(int(m) for m in modes)
        self.eps = float(eps)
        self.w = max(2, math.ceil(math.log10(1.0 / eps)) + 2)          # :255
        self.mrs, self.taus, self.kers = [], [], []
        for m in self.modes:
            mr = next_fast_len(max(2 * m, 2 * self.w + 2))              # :260
            ratio = mr / m
            tau = math.pi * self.w / (ratio * (ratio - 0.5) * m * m)    # :263-264
            h = 2.0 * math.pi / mr
            k = np.arange(m) - m // 2
            j = np.arange(1, self.w + 1)
            ker = 1.0 + 2.0 * (np.exp(-(j * h) ** 2 / (4.0 * tau))[None, :]
                               * np.cos(np.outer(k, j * h))).sum(axis=1)  # :265-270
            self.mrs.append(mr)
            self.taus.append(tau)
            self.kers.append(ker)

    def slots(self):
        return [(np.arange(m) - m // 2) % mr for m, mr in zip(self.modes, self.mrs)]

    def stencils(self, pts):
        """Per-axis fine-grid indices [L, 2w+1] and weights (spectral.py:281-303)."""
        d = len(self.modes)
        offs = np.arange(-self.w, self.w + 1)
        idx, win = [], []
        for a in range(d):
            x = pts[:, d - 1 - a]
            mr, tau = self.mrs[a], self.taus[a]
            h = 2.0 * math.pi / mr
            xi = x - 2.0 * math.pi * np.floor(x / (2.0 * math.pi))
            i0 = np.floor(xi / h + 0.5).astype(np.int64)
            g = i0[:, None] + offs[None, :]
            dl = g * h - xi[:, None]
            idx.append(g % mr)
            win.append(np.exp(-dl * dl / (4.0 * tau)))
        return idx, win


def _outer(arrs):
    return reduce(np.multiply.outer, arrs)


def _check_pts(pts, d):
    pts = np.asarray(pts, dtype=np.float64)
    if pts.ndim == 1:
        pts = pts[:, None]
    _need(pts.ndim == 2 and pts.shape[1] == d and pts.shape[0] >= 1, "bad point array")
    _need(bool(((pts >= -math.pi - 1e-9) & (pts < math.pi + 1e-9)).all()),
          "point coordinates must lie in [-pi, pi)")
    return pts


def _block_weights(win):
    """[L, (2w+1)^d] outer product of the per-axis windows (axis 0 slowest)."""
    out = win[0]
    for wa in win[1:]:
        out = (out[:, :, None] * wa[:, None, :]).reshape(out.shape[0], -1)
    return out


def _block_flat_index(idx, mrs):
    flat = idx[0]
    for ia, mr in zip(idx[1:], mrs[1:]):
        flat = (flat[:, :, None] * mr + ia[:, None, :]).reshape(flat.shape[0], -1)
    return flat


def nufft1(points, values, modes, eps):
    """Type 1, exponent -1j, points -> centred modes (spectral.py:336-358)."""
    plan = NufftPlan(modes, eps)
    pts = _check_pts(points, len(plan.modes))
    vals = np.asarray(values, dtype=np.complex128)
    idx, win = plan.stencils(pts)
    fine = np.zeros(int(np.prod(plan.mrs)), dtype=np.complex128)
    np.add.at(fine, _block_flat_index(idx, plan.mrs).ravel(),
              (vals[:, None] * _block_weights(win)).ravel())
    spec = np.fft.fftn(fine.reshape(plan.mrs))
    return spec[np.ix_(*plan.slots())] / _outer(plan.kers)


def nufft2(coeff, points, eps):
    """Type 2, exponent +1j, centred modes -> points (spectral.py:361-381)."""
    coeff = np.asarray(coeff, dtype=np.complex128)
    plan = NufftPlan(coeff.shape, eps)
    pts = _check_pts(points, coeff.ndim)
    arr = np.zeros(plan.mrs, dtype=np.complex128)
    arr[np.ix_(*plan.slots())] = coeff / _outer(plan.kers)
    fine = (np.fft.ifftn(arr) * float(np.prod(plan.mrs))).ravel()
    idx, win = plan.stencils(pts)
    return (fine[_block_flat_index(idx, plan.mrs)] * _block_weights(win)).sum(axis=1)


def nudft1(points, values, modes):
    """Direct type-1 sum (reference oracle.py:41-53)."""
    pts = np.asarray(points, dtype=np.float64).reshape(len(values), -1)
    d = len(modes)
    grids = np.meshgrid(*[np.arange(m) - m // 2 for m in modes], indexing="ij")
    ph = sum(np.outer(pts[:, d - 1 - a], grids[a].ravel()) for a in range(d))
    return (np.asarray(values) @ np.exp(-1j * ph)).reshape(modes)


def nudft2(coeff, points):
    """Direct type-2 sum (reference oracle.py:56-67)."""
    coeff = np.asarray(coeff, dtype=np.complex128)
    d = coeff.ndim
    pts = np.asarray(points, dtype=np.float64).reshape(-1, d)
    grids = np.meshgrid(*[np.arange(m) - m // 2 for m in coeff.shape], indexing="ij")
    ph = sum(np.outer(pts[:, d - 1 - a], grids[a].ravel()) for a in range(d))
    return np.exp(1j * ph) @ coeff.ravel()


# ---------------------------------------------------------------------------
# shared reconstruction machinery (reference reconstruct.py:90-200)
# ---------------------------------------------------------------------------


def _close(a, b):
    return math.isclose(a, b, rel_tol=1e-9, abs_tol=1e-12)


def _int_offset(value, pitch):
    q = value / pitch
    qi = round(q)
    _need(abs(q - qi) <= 1e-9 * max(1.0, abs(q)), "origin offset must be on the lattice")
    return int(qi)


def pad_size(lag_max, nu_max, n_min):
    """reconstruct.py:102-110."""
    need = 2 * math.ceil(max(lag_max, nu_max)) + 2
    return next_fast_len(max(n_min, need + 8))


def pad_embed(u, py, px):
    """reconstruct.py:113-119 (works on a leading batch axis too)."""
    ny, nx = u.shape[-2:]
    out = np.zeros(u.shape[:-2] + (py, px), dtype=np.complex128)
    oy, ox = py // 2 - ny // 2, px // 2 - nx // 2
    out[..., oy:oy + ny, ox:ox + nx] = u
    return out


def center_slice(p, n):
    """reconstruct.py:122-125."""
    s = p // 2 - n // 2
    return slice(s, s + n)


def kernel_2d(khat, lag_x, lag_y, dz):
    """``exp(+1j k r)/r`` on the lag lattice (reconstruct.py:128-130)."""
    r = np.sqrt(lag_x[None, :] ** 2 + lag_y[:, None] ** 2 + dz * dz)
    return np.exp(SIGN * 1j * khat * r) / r


def illum_mask(khat, xs, ys, z, src):
    """reconstruct.py:133-137."""
    r = np.sqrt((xs[None, :] - src[0]) ** 2 + (ys[:, None] - src[1]) ** 2 + (z - src[2]) ** 2)
    return np.exp(SIGN * 1j * khat * r)


def illum_phase_points(khat, pts_xy, z, src):
    """reconstruct.py:140-144."""
    r = np.sqrt((pts_xy[:, 0] - src[0]) ** 2 + (pts_xy[:, 1] - src[1]) ** 2 + (z - src[2]) ** 2)
    return np.exp(SIGN * 1j * khat * r)


def ill_coords(slices):
    """reference core.py:255-261."""
    il = slices.illuminations
    pts = np.asarray(il.points, dtype=np.float64)
    if pts.shape[1] == 3:
        return pts
    return np.column_stack([pts, np.full(len(pts), float(slices.relay.z))])


def _reduce(terms, freqs, count, times):
    """Ascending-frequency sum; frames weight each term by exp(1j w t) (reconstruct.py:163-177)."""
    if times is None:
        out = np.zeros(count, dtype=np.complex128)
        for term in terms:
            out += term
        return out
    t = np.asarray(times, dtype=np.float64)
    frames = np.zeros((t.size, count), dtype=np.complex128)
    for fi, term in enumerate(terms):
        for ti in range(t.size):
            frames[ti] += np.exp(1j * float(freqs[fi]) * t[ti]) * term
    return frames


def _chunks(n, size):
    for s in range(0, n, size):
        yield s, min(n, s + size)


def _propagate_planes(uhat, khat, lag_x, lag_y, dzs, rows, cols, plane_xy, plane_z,
                      src, include_ill, chunk=8):
    """cifft2(uhat * cfft2(G_k))[rows, cols] (* mask) for every plane k, batched."""
    out = []
    for a, b in _chunks(len(dzs), chunk):
        g = np.stack([kernel_2d(khat, lag_x[k] if isinstance(lag_x, list) else lag_x,
                                lag_y[k] if isinstance(lag_y, list) else lag_y, dzs[k])
                      for k in range(a, b)])
        u = uhat if uhat.ndim == 2 else uhat[a:b]
        planes = cifft2(u * cfft2(g))[:, rows, cols]
        if include_ill:
            for i, k in enumerate(range(a, b)):
                xs, ys = plane_xy(k)
                planes[i] = planes[i] * illum_mask(khat, xs, ys, plane_z(k), src)
        out.append(planes)
    return np.concatenate(out, axis=0)


# ---------------------------------------------------------------------------
# algorithms (reference reconstruct.py:208-765)
# ---------------------------------------------------------------------------


def rsd(slices, grid, padding="exact", times=None, include_illumination=True,
        plane_range=None, freq_range=None):
    """Uniform relay -> cuboid at the relay pitch (reconstruct.py:208-268).

    ``plane_range``/``freq_range`` restrict the work to a subset (used for the
    bounded CPU-baseline samples; every (f, k) unit is independent).
    """
    _need(slices.relay.kind == "uniform", "rsd needs a uniform relay")
    g = slices.relay.grid
    vg = grid.grid
    _need(_close(vg.dx, g.dx) and _close(vg.dy, g.dy), "output lateral pitch must equal the relay pitch")
    cx, cy = g.center()
    nu0x = _int_offset(vg.x0 - cx, g.dx)
    nu0y = _int_offset(vg.y0 - cy, g.dy)
    nux = nu0x + np.arange(vg.nx)
    nuy = nu0y + np.arange(vg.ny)
    zs = vg.z_coords()
    jx_lo, jx_hi = -(g.nx // 2), g.nx - g.nx // 2 - 1
    jy_lo, jy_hi = -(g.ny // 2), g.ny - g.ny // 2 - 1
    if padding == "none":
        px, py = g.nx, g.ny
    else:
        lx = max(abs(int(nux.min()) - jx_hi), abs(int(nux.max()) - jx_lo))
        ly = max(abs(int(nuy.min()) - jy_hi), abs(int(nuy.max()) - jy_lo))
        px = pad_size(lx, max(abs(int(nux.min())), abs(int(nux.max())), g.nx // 2), g.nx)
        py = pad_size(ly, max(abs(int(nuy.min())), abs(int(nuy.max())), g.ny // 2), g.ny)
    lag_x = (np.arange(px) - px // 2) * g.dx
    lag_y = (np.arange(py) - py // 2) * g.dy
    ill = ill_coords(slices)
    xs = vg.x0 + vg.dx * np.arange(vg.nx)
    ys = vg.y0 + vg.dy * np.arange(vg.ny)
    rows = (py // 2 + nuy)[:, None]
    cols = (px // 2 + nux)[None, :]
    k_lo, k_hi = plane_range or (0, zs.size)
    f_lo, f_hi = freq_range or (0, slices.n_freq)
    coeff = np.asarray(slices.coefficients)
    freqs = np.asarray(slices.frequencies)

    def term(fi):
        khat = freqs[fi] / C
        vol = np.zeros((k_hi - k_lo, vg.ny, vg.nx), dtype=np.complex128)
        for p in range(ill.shape[0]):
            uhat = cfft2(pad_embed(coeff[p, :, fi].reshape(g.ny, g.nx), py, px))
            vol += _propagate_planes(uhat, khat, lag_x, lag_y, zs[k_lo:k_hi] - g.z,
                                     rows, cols, lambda k: (xs, ys),
                                     lambda k: float(zs[k_lo + k]), ill[p],
                                     include_illumination)
        return vol.ravel()

    count = (k_hi - k_lo) * vg.ny * vg.nx
    return _reduce((term(f) for f in range(f_lo, f_hi)), freqs[f_lo:f_hi], count, times)


def srsd(slices, grid, times=None, include_illumination=True, plane_range=None,
         freq_range=None):
    """Uniform relay -> depth-scaled frustum (reconstruct.py:276-327)."""
    _need(slices.relay.kind == "uniform", "srsd needs a uniform relay")
    g = slices.relay.grid
    px = next_fast_len(2 * g.nx)
    py = next_fast_len(2 * g.ny)
    rows = center_slice(py, g.ny)
    cols = center_slice(px, g.nx)
    ill = ill_coords(slices)
    coeff = np.asarray(slices.coefficients)
    freqs = np.asarray(slices.frequencies)
    k_lo, k_hi = plane_range or (0, grid.n_planes)
    f_lo, f_hi = freq_range or (0, slices.n_freq)
    ks = list(range(k_lo, k_hi))
    al = [float(grid.alphas[k]) for k in ks]
    be = [float(grid.betas[k]) for k in ks]
    lxs = [(np.arange(px) - px // 2) * (g.dx / a) for a in al]
    lys = [(np.arange(py) - py // 2) * (g.dy / b) for b in be]
    dzs = np.asarray([float(grid.zs[k]) - g.z for k in ks])

    def term(fi):
        khat = freqs[fi] / C
        vol = np.zeros((len(ks), g.ny, g.nx), dtype=np.complex128)
        for p in range(ill.shape[0]):
            u_pad = pad_embed(coeff[p, :, fi].reshape(g.ny, g.nx), py, px)
            uh = np.stack([sfft_2d_centered(u_pad, a, b) for a, b in zip(al, be)])
            vol += _propagate_planes(uh, khat, lxs, lys, dzs, rows, cols,
                                     lambda i: grid.plane_xy(ks[i]),
                                     lambda i: float(grid.zs[ks[i]]), ill[p],
                                     include_illumination)
        return vol.ravel()

    count = len(ks) * g.ny * g.nx
    return _reduce((term(f) for f in range(f_lo, f_hi)), freqs[f_lo:f_hi], count, times)


def nursd1_geometry(slices, grid):
    """Pad sizes and torus coordinates of nursd1 (reconstruct.py:345-361)."""
    vg = grid.grid
    cx = vg.x0 + (vg.nx // 2) * vg.dx
    cy = vg.y0 + (vg.ny // 2) * vg.dy
    rel = np.asarray(slices.relay.points.points)
    nu_rx = (rel[:, 0] - cx) / vg.dx
    nu_ry = (rel[:, 1] - cy) / vg.dy
    lo_x, hi_x = -(vg.nx // 2), vg.nx - vg.nx // 2 - 1
    lo_y, hi_y = -(vg.ny // 2), vg.ny - vg.ny // 2 - 1
    lx = max(hi_x - nu_rx.min(), nu_rx.max() - lo_x)
    ly = max(hi_y - nu_ry.min(), nu_ry.max() - lo_y)
    px = pad_size(lx, max(abs(nu_rx).max(), vg.nx // 2), vg.nx)
    py = pad_size(ly, max(abs(nu_ry).max(), vg.ny // 2), vg.ny)
    torus = np.column_stack([2.0 * np.pi * nu_rx / px, 2.0 * np.pi * nu_ry / py])
    return px, py, torus


def nursd1(slices, grid, eps=1e-6, times=None, include_illumination=True,
           plane_range=None, freq_range=None):
    """Scattered planar relay -> cuboid (reconstruct.py:335-385)."""
    _need(slices.relay.kind == "nonuniform_planar", "nursd1 needs a scattered planar relay")
    vg = grid.grid
    zs = vg.z_coords()
    px, py, torus = nursd1_geometry(slices, grid)
    rows = center_slice(py, vg.ny)
    cols = center_slice(px, vg.nx)
    lag_x = (np.arange(px) - px // 2) * vg.dx
    lag_y = (np.arange(py) - py // 2) * vg.dy
    ill = ill_coords(slices)
    xs = vg.x0 + vg.dx * np.arange(vg.nx)
    ys = vg.y0 + vg.dy * np.arange(vg.ny)
    coeff = np.asarray(slices.coefficients)
    freqs = np.asarray(slices.frequencies)
    k_lo, k_hi = plane_range or (0, zs.size)
    f_lo, f_hi = freq_range or (0, slices.n_freq)
    z_rel = float(slices.relay.z)

    def term(fi):
        khat = freqs[fi] / C
        vol = np.zeros((k_hi - k_lo, vg.ny, vg.nx), dtype=np.complex128)
        for p in range(ill.shape[0]):
            uhat = nufft1(torus, coeff[p, :, fi], (py, px), eps)
            vol += _propagate_planes(uhat, khat, lag_x, lag_y, zs[k_lo:k_hi] - z_rel,
                                     rows, cols, lambda k: (xs, ys),
                                     lambda k: float(zs[k_lo + k]), ill[p],
                                     include_illumination)
        return vol.ravel()

    count = (k_hi - k_lo) * vg.ny * vg.nx
    return _reduce((term(f) for f in range(f_lo, f_hi)), freqs[f_lo:f_hi], count, times)


def _explicit_geo(grid, cx, cy, dx, dy, sx=1.0, sy=1.0):
    """reconstruct.py:393-410."""
    geo, start = [], 0
    for pl in grid.planes:
        pts = np.asarray(pl.points.points)
        geo.append((start, pts.shape[0], sx * (pts[:, 0] - cx) / dx,
                    sy * (pts[:, 1] - cy) / dy, pts, float(pl.z)))
        start += pts.shape[0]
    return geo


def _explicit_run(slices, grid, geo, px, py, lag_x, lag_y, z_rel, uhat_of, eps, times,
                  include_illumination):
    """Shared per-plane type-2 readout of nursd2/nursd3/srsd_nursd2."""
    toruses = [np.column_stack([2.0 * np.pi * t[2] / px, 2.0 * np.pi * t[3] / py]) for t in geo]
    ill = ill_coords(slices)
    freqs = np.asarray(slices.frequencies)
    scale = 1.0 / (px * py)

    def term(fi):
        khat = freqs[fi] / C
        vol = np.zeros(grid.count, dtype=np.complex128)
        for p in range(ill.shape[0]):
            uhat = uhat_of(p, fi)
            for k, (start, cnt, _, _, pts, z) in enumerate(geo):
                gh = cfft2(kernel_2d(khat, lag_x, lag_y, z - z_rel))
                vals = nufft2(uhat * gh, toruses[k], eps) * scale
                if include_illumination:
                    vals = vals * illum_phase_points(khat, pts, z, ill[p])
                vol[start:start + cnt] += vals
        return vol

    return _reduce((term(f) for f in range(slices.n_freq)), freqs, grid.count, times)


def nursd2(slices, grid, eps=1e-6, times=None, include_illumination=True):
    """Uniform relay -> explicit voxels (reconstruct.py:413-459)."""
    _need(slices.relay.kind == "uniform", "nursd2 needs a uniform relay")
    g = slices.relay.grid
    cx, cy = g.center()
    geo = _explicit_geo(grid, cx, cy, g.dx, g.dy)
    jx_lo, jx_hi = -(g.nx // 2), g.nx - g.nx // 2 - 1
    jy_lo, jy_hi = -(g.ny // 2), g.ny - g.ny // 2 - 1
    ax = np.concatenate([t[2] for t in geo])
    ay = np.concatenate([t[3] for t in geo])
    lx = max(ax.max() - jx_lo, jx_hi - ax.min())
    ly = max(ay.max() - jy_lo, jy_hi - ay.min())
    px = pad_size(lx, max(abs(ax).max(), g.nx // 2), g.nx)
    py = pad_size(ly, max(abs(ay).max(), g.ny // 2), g.ny)
    lag_x = (np.arange(px) - px // 2) * g.dx
    lag_y = (np.arange(py) - py // 2) * g.dy
    coeff = np.asarray(slices.coefficients)

    def uhat_of(p, fi):
        return cfft2(pad_embed(coeff[p, :, fi].reshape(g.ny, g.nx), py, px))

    return _explicit_run(slices, grid, geo, px, py, lag_x, lag_y, g.z, uhat_of, eps, times,
                         include_illumination)


def nursd3(slices, grid, eps=1e-6, lattice_pitch=None, times=None, include_illumination=True):
    """Scattered planar relay -> explicit voxels via a virtual lattice (reconstruct.py:467-525)."""
    _need(slices.relay.kind == "nonuniform_planar", "nursd3 needs a scattered planar relay")
    pitch = float(lattice_pitch) if lattice_pitch is not None else slices.shortest_wavelength / 2.0
    _need(pitch > 0, "lattice pitch must be > 0")
    rel = np.asarray(slices.relay.points.points)
    tgt = np.vstack([np.asarray(p.points.points) for p in grid.planes])
    lo = np.minimum(rel.min(axis=0), tgt.min(axis=0))
    hi = np.maximum(rel.max(axis=0), tgt.max(axis=0))
    anchor = rel[0] + np.round(((lo + hi) / 2.0 - rel[0]) / pitch) * pitch
    cx, cy = float(anchor[0]), float(anchor[1])
    nu_rx = (rel[:, 0] - cx) / pitch
    nu_ry = (rel[:, 1] - cy) / pitch
    geo = _explicit_geo(grid, cx, cy, pitch, pitch)
    ax = np.concatenate([t[2] for t in geo])
    ay = np.concatenate([t[3] for t in geo])
    lx = max(ax.max() - nu_rx.min(), nu_rx.max() - ax.min())
    ly = max(ay.max() - nu_ry.min(), nu_ry.max() - ay.min())
    px = pad_size(lx, max(abs(ax).max(), abs(nu_rx).max()), 1)
    py = pad_size(ly, max(abs(ay).max(), abs(nu_ry).max()), 1)
    torus_rel = np.column_stack([2.0 * np.pi * nu_rx / px, 2.0 * np.pi * nu_ry / py])
    lag_x = (np.arange(px) - px // 2) * pitch
    lag_y = (np.arange(py) - py // 2) * pitch
    coeff = np.asarray(slices.coefficients)

    def uhat_of(p, fi):
        return nufft1(torus_rel, coeff[p, :, fi], (py, px), eps)

    return _explicit_run(slices, grid, geo, px, py, lag_x, lag_y, float(slices.relay.z),
                         uhat_of, eps, times, include_illumination)


def srsd_nursd2(slices, grid, alpha, beta=None, eps=1e-6, times=None,
                include_illumination=True):
    """Uniform relay -> explicit voxels through one scaled transform (reconstruct.py:533-586)."""
    beta = alpha if beta is None else beta
    _need(0 < alpha <= 1 and 0 < beta <= 1, "scale factors must lie in (0, 1]")
    g = slices.relay.grid
    cx, cy = g.center()
    geo = _explicit_geo(grid, cx, cy, g.dx, g.dy, alpha, beta)
    jx_lo, jx_hi = -(g.nx // 2), g.nx - g.nx // 2 - 1
    jy_lo, jy_hi = -(g.ny // 2), g.ny - g.ny // 2 - 1
    ax = np.concatenate([t[2] for t in geo])
    ay = np.concatenate([t[3] for t in geo])
    lx = max(ax.max() - alpha * jx_lo, alpha * jx_hi - ax.min())
    ly = max(ay.max() - beta * jy_lo, beta * jy_hi - ay.min())
    px = pad_size(lx, max(abs(ax).max(), g.nx // 2), g.nx)
    py = pad_size(ly, max(abs(ay).max(), g.ny // 2), g.ny)
    lag_x = (np.arange(px) - px // 2) * (g.dx / alpha)
    lag_y = (np.arange(py) - py // 2) * (g.dy / beta)
    coeff = np.asarray(slices.coefficients)

    def uhat_of(p, fi):
        return sfft_2d_centered(pad_embed(coeff[p, :, fi].reshape(g.ny, g.nx), py, px),
                                alpha, beta)

    return _explicit_run(slices, grid, geo, px, py, lag_x, lag_y, g.z, uhat_of, eps, times,
                         include_illumination)


def lattice_3d(slices, grid, z_pitch=None):
    """Virtual 3D lattice geometry (reconstruct.py:594-621)."""
    vg = grid.grid
    rel = np.asarray(slices.relay.points.points)
    dz3 = float(z_pitch) if z_pitch else slices.shortest_wavelength / 2.0
    z_min = float(rel[:, 2].min())
    nz3 = max(1, math.ceil((float(rel[:, 2].max()) - z_min) / dz3) + 1)
    pz = next_fast_len(2 * nz3 + 2)
    z0 = z_min + nz3 * dz3
    _need(bool((vg.z_coords() > z0).all()), "every voxel plane must lie beyond the far face")
    cx = vg.x0 + (vg.nx // 2) * vg.dx
    cy = vg.y0 + (vg.ny // 2) * vg.dy
    nu_rx = (rel[:, 0] - cx) / vg.dx
    nu_ry = (rel[:, 1] - cy) / vg.dy
    lo_x, hi_x = -(vg.nx // 2), vg.nx - vg.nx // 2 - 1
    lo_y, hi_y = -(vg.ny // 2), vg.ny - vg.ny // 2 - 1
    lx = max(hi_x - nu_rx.min(), nu_rx.max() - lo_x)
    ly = max(hi_y - nu_ry.min(), nu_ry.max() - lo_y)
    px = pad_size(lx, max(abs(nu_rx).max(), vg.nx // 2), vg.nx)
    py = pad_size(ly, max(abs(nu_ry).max(), vg.ny // 2), vg.ny)
    slab = pz // 2 + (nz3 - nz3 // 2)
    return dict(rel=rel, dz3=dz3, z_min=z_min, nz3=nz3, pz=pz, z0=z0, nu_rx=nu_rx,
                nu_ry=nu_ry, px=px, py=py, slab=slab)


def kernel_3d(khat, px, py, pz, dx, dy, dz3):
    """3D kernel with the zero-lag slot zeroed (reconstruct.py:624-638)."""
    lx = (np.arange(px) - px // 2) * dx
    ly = (np.arange(py) - py // 2) * dy
    lz = (np.arange(pz) - pz // 2) * dz3
    r = np.sqrt(lz[:, None, None] ** 2 + ly[None, :, None] ** 2 + lx[None, None, :] ** 2)
    c = (pz // 2, py // 2, px // 2)
    r[c] = 1.0
    k = np.exp(SIGN * 1j * khat * r) / r
    k[c] = 0.0
    return k


def nursd3d_stage1(slices, grid, eps=1e-6, z_pitch=None):
    """Per (f, illumination) virtual-plane spectrum ``cfft2(wave[slab])`` (reconstruct.py:741-760).

    Returns (geometry dict, list over f of [I, py, px] arrays).
    """
    geo = lattice_3d(slices, grid, z_pitch)
    vg = grid.grid
    c_z = geo["z_min"] + (geo["nz3"] // 2) * geo["dz3"]
    nu_rz = (geo["rel"][:, 2] - c_z) / geo["dz3"]
    px, py, pz = geo["px"], geo["py"], geo["pz"]
    torus = np.column_stack([2.0 * np.pi * geo["nu_rx"] / px, 2.0 * np.pi * geo["nu_ry"] / py,
                             2.0 * np.pi * nu_rz / pz])
    coeff = np.asarray(slices.coefficients)
    out = []
    for fi, w in enumerate(np.asarray(slices.frequencies)):
        khat = w / C
        g3 = cfft(kernel_3d(khat, px, py, pz, vg.dx, vg.dy, geo["dz3"]), (-3, -2, -1))
        per_p = []
        for p in range(coeff.shape[0]):
            u3 = nufft1(torus, coeff[p, :, fi], (pz, py, px), eps)
            wave = cifft(u3 * g3, (-3, -2, -1))
            per_p.append(cfft2(wave[geo["slab"]]))
        out.append(np.stack(per_p))
    return geo, out


def rsd3d_scatter(geo, scatter):
    """Lattice slots and weights of the stage-1 gridding (reconstruct.py:680-703): nearest
    (1 slot, weight 1) or trilinear (8 corners, products of the per-axis linear weights);
    slot index j on an axis of length n is the centred lag j - n//2."""
    px, py, pz = geo["px"], geo["py"], geo["pz"]
    fx = geo["nu_rx"] + px // 2
    fy = geo["nu_ry"] + py // 2
    fz = (geo["rel"][:, 2] - geo["z_min"]) / geo["dz3"] + (pz // 2 - geo["nz3"] // 2)
    if scatter == "nearest":
        ix = np.round(fx).astype(np.int64)[:, None]
        iy = np.round(fy).astype(np.int64)[:, None]
        iz = np.round(fz).astype(np.int64)[:, None]
        w = np.ones((fx.size, 1))
    else:
        def corners(f):
            lo = np.floor(f).astype(np.int64)
            fr = f - lo
            return np.stack([lo, lo + 1], axis=1), np.stack([1.0 - fr, fr], axis=1)
        gx, wx = corners(fx)
        gy, wy = corners(fy)
        gz, wz = corners(fz)
        iz = np.broadcast_to(gz[:, :, None, None], (fx.size, 2, 2, 2)).reshape(-1, 8)
        iy = np.broadcast_to(gy[:, None, :, None], (fx.size, 2, 2, 2)).reshape(-1, 8)
        ix = np.broadcast_to(gx[:, None, None, :], (fx.size, 2, 2, 2)).reshape(-1, 8)
        w = (wz[:, :, None, None] * wy[:, None, :, None] * wx[:, None, None, :]).reshape(-1, 8)
    for idx, n in ((ix, px), (iy, py), (iz, pz)):
        _need(idx.min() >= 0 and idx.max() < n, "relay scatter indices escaped the lattice")
    return iz, iy, ix, w


def rsd3d_stage1(slices, grid, scatter="trilinear", z_pitch=None):
    """Per (f, illumination) virtual-plane spectrum of rsd3d (reconstruct.py:705-716):
    gridding, cfft_n, x cfft_n(G3), cifft_n, slab, cfft_2d."""
    geo = lattice_3d(slices, grid, z_pitch)
    vg = grid.grid
    px, py, pz = geo["px"], geo["py"], geo["pz"]
    iz, iy, ix, w = rsd3d_scatter(geo, scatter)
    coeff = np.asarray(slices.coefficients)
    out = []
    for fi, om in enumerate(np.asarray(slices.frequencies)):
        khat = om / C
        g3 = cfft(kernel_3d(khat, px, py, pz, vg.dx, vg.dy, geo["dz3"]), (-3, -2, -1))
        per_p = []
        for p in range(coeff.shape[0]):
            fine = np.zeros((pz, py, px), dtype=np.complex128)
            np.add.at(fine, (iz, iy, ix), coeff[p, :, fi][:, None] * w)
            wave = cifft(cfft(fine, (-3, -2, -1)) * g3, (-3, -2, -1))
            per_p.append(cfft2(wave[geo["slab"]]))
        out.append(np.stack(per_p))
    return geo, out


def rsd3d(slices, grid, scatter="trilinear", z_pitch=None, times=None,
          include_illumination=True):
    """3D relay -> cuboid by gridding + 3D convolution (reconstruct.py:662-719)."""
    geo, uplanes = rsd3d_stage1(slices, grid, scatter, z_pitch)
    return _stage2(slices, grid, geo, uplanes, times, include_illumination)


def _stage2(slices, grid, geo, uplanes, times, include_illumination):
    """Virtual plane z0 -> every output plane (reconstruct.py:641-659)."""
    vg = grid.grid
    px, py = geo["px"], geo["py"]
    zs = vg.z_coords()
    lag_x = (np.arange(px) - px // 2) * vg.dx
    lag_y = (np.arange(py) - py // 2) * vg.dy
    rows = center_slice(py, vg.ny)
    cols = center_slice(px, vg.nx)
    xs = vg.x0 + vg.dx * np.arange(vg.nx)
    ys = vg.y0 + vg.dy * np.arange(vg.ny)
    ill = ill_coords(slices)
    freqs = np.asarray(slices.frequencies)

    def term(fi):
        khat = freqs[fi] / C
        vol = np.zeros((zs.size, vg.ny, vg.nx), dtype=np.complex128)
        for p in range(ill.shape[0]):
            vol += _propagate_planes(uplanes[fi][p], khat, lag_x, lag_y, zs - geo["z0"],
                                     rows, cols, lambda k: (xs, ys), lambda k: float(zs[k]),
                                     ill[p], include_illumination)
        return vol.ravel()

    return _reduce((term(f) for f in range(slices.n_freq)), freqs, grid.count, times)


def nursd3d(slices, grid, eps=1e-6, z_pitch=None, times=None, include_illumination=True):
    """3D scattered relay -> cuboid (reconstruct.py:722-765)."""
    rel = np.asarray(slices.relay.points.points)
    if float(rel[:, 2].max() - rel[:, 2].min()) == 0.0:
        flat = _FlatView(slices, rel)
        return nursd1(flat, grid, eps=eps, times=times,
                      include_illumination=include_illumination)
    geo, uplanes = nursd3d_stage1(slices, grid, eps, z_pitch)
    vg = grid.grid
    px, py = geo["px"], geo["py"]
    zs = vg.z_coords()
    lag_x = (np.arange(px) - px // 2) * vg.dx
    lag_y = (np.arange(py) - py // 2) * vg.dy
    rows = center_slice(py, vg.ny)
    cols = center_slice(px, vg.nx)
    xs = vg.x0 + vg.dx * np.arange(vg.nx)
    ys = vg.y0 + vg.dy * np.arange(vg.ny)
    ill = ill_coords(slices)
    freqs = np.asarray(slices.frequencies)

    def term(fi):
        khat = freqs[fi] / C
        vol = np.zeros((zs.size, vg.ny, vg.nx), dtype=np.complex128)
        for p in range(ill.shape[0]):
            vol += _propagate_planes(uplanes[fi][p], khat, lag_x, lag_y, zs - geo["z0"],
                                     rows, cols, lambda k: (xs, ys), lambda k: float(zs[k]),
                                     ill[p], include_illumination)
        return vol.ravel()

    return _reduce((term(f) for f in range(slices.n_freq)), freqs, grid.count, times)


def nursd3d_explicit(slices, grid, lattice, eps=1e-6, z_pitch=None, times=None,
                     include_illumination=True):
    """Config-2 composed oracle: nursd3d stage 1 to the virtual plane z0
    (reconstruct.py:741-760), then nursd2 (:413-459) from a uniform relay at z0 that
    carries that plane's centred-slot coefficients."""
    geo, uplanes = nursd3d_stage1(slices, lattice, eps, z_pitch)
    vg = lattice.grid
    px, py = geo["px"], geo["py"]
    cx = vg.x0 + (vg.nx // 2) * vg.dx
    cy = vg.y0 + (vg.ny // 2) * vg.dy
    waves = [cifft2(u) for u in uplanes]                 # [I, py, px] per f, slot order
    coeff = np.stack([w.reshape(w.shape[0], -1) for w in waves], axis=-1)   # [I, D, F]
    grid2 = type("G", (), dict(nx=px, ny=py, dx=vg.dx, dy=vg.dy, x0=cx - (px // 2) * vg.dx,
                              y0=cy - (py // 2) * vg.dy, z=geo["z0"],
                              center=lambda self: (cx, cy)))()
    relay = type("R", (), dict(kind="uniform", grid=grid2, z=geo["z0"], count=px * py))()
    vs = type("S", (), dict(frequencies=slices.frequencies, coefficients=coeff, relay=relay,
                            illuminations=slices.illuminations,
                            n_freq=int(np.asarray(slices.frequencies).size)))()
    return nursd2(vs, grid, eps=eps, times=times, include_illumination=include_illumination)


def lattice_srsd(slices, frustum, stage1="nursd3d", eps=1e-6, scatter="trilinear",
                 z_pitch=None, times=None, include_illumination=True):
    """Composed oracle of the paper's "3D RSD / 3D NURSD + SRSD":
    nursd3d stage 1 (reconstruct.py:741-760) or rsd3d stage 1 (:705-716) on the lattice of
    the frustum base, the wave slab at z0 cropped to the base window (the centred rows /
    columns of reconstruct.py:650-651), then srsd (:276-327) from that uniform relay at z0."""
    b = frustum.base
    zs = np.asarray(frustum.zs, dtype=np.float64)
    vg = type("G", (), dict(nx=b.nx, ny=b.ny, dx=b.dx, dy=b.dy, x0=b.x0, y0=b.y0,
                            z_coords=lambda self: zs))()
    lattice = type("L", (), dict(grid=vg))()
    if stage1 == "nursd3d":
        geo, uplanes = nursd3d_stage1(slices, lattice, eps, z_pitch)
    else:
        geo, uplanes = rsd3d_stage1(slices, lattice, scatter, z_pitch)
    rows = center_slice(geo["py"], b.ny)
    cols = center_slice(geo["px"], b.nx)
    waves = [cifft2(u)[:, rows, cols] for u in uplanes]          # [I, ny, nx] per f
    coeff = np.stack([w.reshape(w.shape[0], -1) for w in waves], axis=-1)   # [I, D, F]
    grid2 = type("G2", (), dict(nx=b.nx, ny=b.ny, dx=b.dx, dy=b.dy, x0=b.x0, y0=b.y0,
                                z=geo["z0"], center=lambda self: (
                                    b.x0 + (b.nx // 2) * b.dx, b.y0 + (b.ny // 2) * b.dy)))()
    relay = type("R", (), dict(kind="uniform", grid=grid2, z=geo["z0"], count=b.nx * b.ny))()
    vs = type("S", (), dict(frequencies=slices.frequencies, coefficients=coeff, relay=relay,
                            illuminations=slices.illuminations,
                            n_freq=int(np.asarray(slices.frequencies).size)))()
    return srsd(vs, frustum, times=times, include_illumination=include_illumination)


class _FlatView:
    """A 3D relay whose points share one z, viewed as a planar relay (reconstruct.py:735-740)."""

    class _Relay:
        kind = "nonuniform_planar"

        def __init__(self, rel):
            self.points = type("P", (), {"points": rel[:, :2]})()
            self.z = float(rel[0, 2])
            self.count = rel.shape[0]

    def __init__(self, slices, rel):
        self.frequencies = slices.frequencies
        self.coefficients = slices.coefficients
        self.illuminations = slices.illuminations
        self.n_freq = slices.n_freq
        self.relay = self._Relay(rel)


# ---------------------------------------------------------------------------
# exact-physics checker and projections
# ---------------------------------------------------------------------------


def literal_field(slices, voxels, include_illumination=True):
    """Per-voxel 1/r sum the fast propagators evaluate (reference tests/helpers.py:69-101)."""
    det = np.asarray(slices.relay.coordinates())
    ill = ill_coords(slices)
    vox = np.asarray(voxels, dtype=np.float64)
    coeff = np.asarray(slices.coefficients)
    out = np.zeros(vox.shape[0], dtype=np.complex128)
    for vi, v in enumerate(vox):
        r_det = np.sqrt(((det - v) ** 2).sum(axis=1))
        r_ill = np.sqrt(((ill - v) ** 2).sum(axis=1))
        acc = 0.0 + 0.0j
        for fi, w in enumerate(np.asarray(slices.frequencies)):
            kh = w / C
            kern = np.exp(SIGN * 1j * kh * r_det) / r_det
            for p in range(ill.shape[0]):
                t = np.sum(coeff[p, :, fi] * kern)
                if include_illumination:
                    t = t * np.exp(SIGN * 1j * kh * r_ill[p])
                acc += t
        out[vi] = acc
    return out


def project_max_depth(field3d):
    """``max_z |field|`` (reconstruct.py:834-836)."""
    return np.abs(field3d).max(axis=0)


def rel_l2(a, b):
    d = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / d) if d else float(np.linalg.norm(a - b))


def rel_linf(a, b):
    d = np.max(np.abs(b))
    return float(np.max(np.abs(a - b)) / d) if d else float(np.max(np.abs(a - b)))
