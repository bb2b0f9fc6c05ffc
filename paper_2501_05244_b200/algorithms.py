"""GPU drop-ins for srsd, nursd1, nursd2, nursd3, srsd_nursd2, nursd3d (reference reconstruct.py).

Host code computes sizes exactly as the reference does (the pad rules decide the
result wherever the relay or the voxels sit off the lattice: SURVEY F2/F3) and
drives the ``libpfgpu`` kernels: Bluestein lines (srsd), NUFFT type 1
(nursd1/3, nursd3d stage 1), the propagation kernels A/B/C, and the type-2
readout (product -> place -> inverse FFT -> interpolate+accumulate).
"""

from __future__ import annotations

import ctypes
import math
import os

import numpy as np
import torch

from . import _device as dev
from . import _lib
from . import nufft as nu
from ._fastlen import next_fast_len
from .core import SPEED_OF_LIGHT, _require
from .phasor import device_coefficients
from .reconstruct import (GraphedRun, PlaneSpec, Propagator, _check_depths, _check_times, _close,
                          _exact_pad, _frame_weights, _ill_tensor, _kind, _nonplanar_relay,
                          _pad_size, _planar_relay, _uniform_relay, _volume, cached_engine, rsd)

C = SPEED_OF_LIGHT
_BATCH_BYTES = int(os.environ.get("PF_SRSD_BATCH_MB", "96")) << 20
_SRSD_MINQ = int(os.environ.get("PF_SRSD_MINQ", "8"))   # plane multiple (x 32/L)


def _center_nu0(n: int) -> int:
    return -(n // 2)


# ---------------------------------------------------------------------------
# scaled-FFT tables (reference spectral.py:143-158, cached like :171-180)
# ---------------------------------------------------------------------------

_SFFT_TABLES: dict = {}


def _sfft_tables(m: int, alpha: float, offset: int, q: int):
    key = (m, float(alpha), offset, q)
    t = _SFFT_TABLES.get(key)
    if t is None:
        n = np.arange(m, dtype=np.float64) - offset
        chirp = np.exp(-1j * np.pi * alpha * n * n / m)
        lags = np.arange(1 - m, m)
        kern = np.zeros(q, dtype=np.complex128)
        kern[lags % q] = np.exp(1j * np.pi * alpha * lags * lags / m)
        t = (chirp.astype(np.complex64), np.fft.fft(kern).astype(np.complex64))
        _SFFT_TABLES[key] = t
    return t


class _ScaledTables:
    """Per-plane chirps / kernel spectra for both axes, on the device."""

    def __init__(self, mx, my, alphas, betas, device):
        self.qx = next_fast_len(max(1, 2 * mx - 1))
        self.qy = next_fast_len(max(1, 2 * my - 1))
        cx, kx, cy, ky = [], [], [], []
        for a, b in zip(alphas, betas):
            c, k = _sfft_tables(mx, a, mx // 2, self.qx)
            cx.append(c)
            kx.append(k)
            c, k = _sfft_tables(my, b, my // 2, self.qy)
            cy.append(c)
            ky.append(k)
        t = lambda xs: torch.from_numpy(np.ascontiguousarray(np.stack(xs))).to(device)  # noqa: E731
        self.chirp_x, self.khat_x = t(cx), t(kx)
        self.chirp_y, self.khat_y = t(cy), t(ky)
        self.plan_qx = dev.fft_plan(self.qx, device)
        self.plan_qy = dev.fft_plan(self.qy, device)


def _scaled_spectra(coeff_fp: torch.Tensor, ny: int, nx: int, py: int, px: int,
                    tabs: _ScaledTables, t0: int, nb: int, xbuf: torch.Tensor,
                    out: torch.Tensor, out_plane_stride: int, transposed: bool, stream=None):
    """sfft_2d_centered(pad_embed(u), a_k, b_k) for planes t0..t0+nb of the tables.

    x pass over the ny embedded relay rows (zero rows transform to zero), written
    with natural column order; y pass over all px columns into natural-order
    spectra (reference spectral.py:196-218, reconstruct.py:318-320).
    """
    s = dev.stream_ptr(stream)
    csz = 8
    if transposed and tabs.qx in (128, 256, 512, 1024) and tabs.qy in (128, 256, 512, 1024):
        # register-FFT passes: x pass stored transposed (xbuf[b][col][iy]), y pass
        # reads contiguous rows of it and writes Uhat^T[b][col][row]
        _lib.call("pf_bluestein_warp", 1, dev.ptr(coeff_fp), 0, nx, nx, px // 2 - nx // 2,
                  dev.ptr(xbuf), px * ny, ny, px, ny, nb, tabs.plan_qx.ref,
                  dev.ptr(tabs.chirp_x) + csz * t0 * px, dev.ptr(tabs.khat_x) + csz * t0 * tabs.qx,
                  s)
        _lib.call("pf_bluestein_warp", 0, dev.ptr(xbuf), px * ny, ny, ny, py // 2 - ny // 2,
                  dev.ptr(out), out_plane_stride, py, py, px, nb, tabs.plan_qy.ref,
                  dev.ptr(tabs.chirp_y) + csz * t0 * py, dev.ptr(tabs.khat_y) + csz * t0 * tabs.qy,
                  s)
        return
    _lib.call("pf_bluestein_lines", dev.ptr(coeff_fp), 0, nx, 1, nx, px // 2 - nx // 2,
              dev.ptr(xbuf), ny * px, px, 1, 1, px, ny, nb, tabs.plan_qx.ref,
              dev.ptr(tabs.chirp_x) + csz * t0 * px, dev.ptr(tabs.khat_x) + csz * t0 * tabs.qx, s)
    if transposed:   # out[b][col][row]
        _lib.call("pf_bluestein_lines", dev.ptr(xbuf), ny * px, 1, px, ny, py // 2 - ny // 2,
                  dev.ptr(out), out_plane_stride, py, 1, 1, py, px, nb, tabs.plan_qy.ref,
                  dev.ptr(tabs.chirp_y) + csz * t0 * py, dev.ptr(tabs.khat_y) + csz * t0 * tabs.qy,
                  s)
    else:            # out[b][row][col]
        _lib.call("pf_bluestein_lines", dev.ptr(xbuf), ny * px, 1, px, ny, py // 2 - ny // 2,
                  dev.ptr(out), out_plane_stride, 1, px, 1, py, px, nb, tabs.plan_qy.ref,
                  dev.ptr(tabs.chirp_y) + csz * t0 * py, dev.ptr(tabs.khat_y) + csz * t0 * tabs.qy,
                  s)


# ---------------------------------------------------------------------------
# srsd: uniform relay -> depth-scaled frustum (reconstruct.py:276-327)
# ---------------------------------------------------------------------------


class SrsdEngine(GraphedRun):
    def __init__(self, slices, grid, include_illumination=True, times=None, device=None,
                 plane_range=None):
        _require(_kind(grid) == "frustum", "srsd reconstructs onto a frustum grid")
        relay = _uniform_relay(slices)
        g = relay.grid
        b = grid.base
        _require(b.nx == g.nx and b.ny == g.ny and _close(b.dx, g.dx) and _close(b.dy, g.dy)
                 and _close(b.x0, g.x0) and _close(b.y0, g.y0),
                 "the frustum base must coincide with the relay lattice")
        _check_depths(grid.zs, g.z)
        self.times = _check_times(times)
        self.device = device or dev.require_cuda()
        # P = next_fast_len(2N): the SRSD result depends on it
        px, py = next_fast_len(2 * g.nx), next_fast_len(2 * g.ny)
        self.px, self.py, self.g, self.grid = px, py, g, grid
        self.freqs = np.asarray(slices.frequencies, dtype=np.float64)
        self.n_illum = int(slices.illuminations.count)
        k_lo, k_hi = plane_range or (0, grid.n_planes)
        self.k_lo, self.k_hi = k_lo, k_hi
        ks = list(range(k_lo, k_hi))
        cx, cy = g.center()
        I = self.n_illum
        planes = []
        tmp = Propagator(self.device, px, py, g.nx, g.ny, 0, 0, I, include_illumination,
                         [PlaneSpec(1, 1, 1, 0, 1, 0, 1, 1)], py * px, batch=1)
        self.transposed = tmp.transposed
        per_plane = 8 * (2 * I * py * px + I * g.ny * px)
        batch = max(1, min(len(ks), _BATCH_BYTES // per_plane))
        if self.transposed:
            q = _SRSD_MINQ * (32 // (px // 32))
            batch = min(len(ks), max(q, (batch // q) * q))
        self.batch = batch
        for i, k in enumerate(ks):
            al, be = float(grid.alphas[k]), float(grid.betas[k])
            pxk, pyk = g.dx / al, g.dy / be
            planes.append(PlaneSpec(float(grid.zs[k]) - g.z, pxk, pyk,
                                    cx - (g.nx // 2) * pxk, pxk, cy - (g.ny // 2) * pyk, pyk,
                                    float(grid.zs[k]), (i % batch) * I * py * px, i))
        self.prop = Propagator(self.device, px, py, g.nx, g.ny, _center_nu0(g.nx),
                               _center_nu0(g.ny), I, include_illumination, planes, py * px,
                               batch=batch)
        self.tabs = _ScaledTables(px, py, [grid.alphas[k] for k in ks],
                                  [grid.betas[k] for k in ks], self.device)
        nl = len(self.prop.lane_streams)
        self.uhat_l = [torch.empty((batch * I * py * px,), dtype=torch.complex64,
                                   device=self.device) for _ in range(nl)]
        self.xbuf_l = [torch.empty((batch * g.ny * px,), dtype=torch.complex64,
                                   device=self.device) for _ in range(nl)]
        self.ill = _ill_tensor(slices, self.device)
        self.frame_w = _frame_weights(self.freqs, self.times, self.device)
        self.n_frames = 1 if self.times is None else self.times.size
        self.n_voxels = len(ks) * g.nx * g.ny

    def run(self, coeff: torch.Tensor, vol=None, stream=None):
        if vol is None:
            vol = torch.zeros((self.n_frames, self.n_voxels), dtype=torch.complex64,
                              device=self.device)
        else:
            vol.zero_()
        g, I, px, py = self.g, self.n_illum, self.px, self.py

        def body(b0, b1, lane, ls):
            nb = b1 - b0
            uhat, xbuf = self.uhat_l[lane], self.xbuf_l[lane]
            order, dk = self.prop.freq_order(self.freqs, self.n_frames)
            for fi in order:
                for p in range(I):
                    _scaled_spectra(coeff[fi, p], g.ny, g.nx, py, px, self.tabs, b0, nb, xbuf,
                                    uhat[p * py * px:], I * py * px, self.transposed, ls)
                khat = float(self.freqs[fi]) / C
                self.prop.run_frequency(dev.ptr(uhat), khat, dev.ptr(self.ill),
                                        dev.ptr(self.frame_w) + 8 * fi * self.n_frames,
                                        self.n_frames, vol, self.n_voxels, plane_lo=b0,
                                        plane_hi=b1, stream=ls, lane=lane,
                                        horner=None if dk is None else (dk, fi, len(order)))

        self.prop.run_batches(body, stream)
        return vol


def srsd(slices, grid, times=None, threads: int = 1, include_illumination: bool = True):
    """Scaled propagation onto a depth-widening frustum (reconstruct.py:276-327)."""
    eng = cached_engine("srsd", slices, grid, (bool(include_illumination),
                                               None if times is None else np.asarray(times)),
                        lambda: SrsdEngine(slices, grid, include_illumination, times))
    return _volume(grid, eng.run_dropin(device_coefficients(slices)), eng.times)


# ---------------------------------------------------------------------------
# nursd1: scattered planar relay -> cuboid (reconstruct.py:335-385)
# ---------------------------------------------------------------------------


class _UhatPropEngine(GraphedRun):
    """Shared tail of nursd1 / nursd3d: per-frequency relay spectra -> propagate."""

    def _setup_prop(self, px, py, vg, z_src, include_illumination, k_range, flags=0):
        zs = vg.z_coords()
        k_lo, k_hi = k_range
        planes = [PlaneSpec(zs[k] - z_src, vg.dx, vg.dy, vg.x0, vg.dx, vg.y0, vg.dy, zs[k], 0,
                            k - k_lo) for k in range(k_lo, k_hi)]
        self.prop = Propagator(self.device, px, py, vg.nx, vg.ny, _center_nu0(vg.nx),
                               _center_nu0(vg.ny), self.n_illum, include_illumination, planes,
                               py * px, n_planes_total=vg.nz)
        self.n_voxels = (k_hi - k_lo) * vg.nx * vg.ny

    def _propagate(self, uhat, vol, stream):
        per_f = self.n_illum * self.py * self.px
        if self.prop.fbatch_ok(self.freqs.size, self.n_frames):
            self.prop.run_fbatch(uhat, per_f, self.freqs, dev.ptr(self.ill), self.frame_w, vol,
                                 stream)
            return vol

        def body(b0, b1, lane, ls):
            order, dk = self.prop.freq_order(self.freqs, self.n_frames)
            for fi in order:
                khat = float(self.freqs[fi]) / C
                self.prop.run_frequency(dev.ptr(uhat) + 8 * fi * per_f, khat, dev.ptr(self.ill),
                                        dev.ptr(self.frame_w) + 8 * fi * self.n_frames,
                                        self.n_frames, vol, self.n_voxels, plane_lo=b0,
                                        plane_hi=b1, stream=ls, lane=lane,
                                        horner=None if dk is None else (dk, fi, len(order)))

        self.prop.run_batches(body, stream)
        return vol


class Nursd1Engine(_UhatPropEngine):
    def __init__(self, slices, grid, eps=1e-6, include_illumination=True, times=None,
                 device=None, plane_range=None):
        _require(_kind(grid) == "cuboid", "nursd1 reconstructs onto a cuboid grid")
        relay = _planar_relay(slices)
        vg = grid.grid
        zs = vg.z_coords()
        _check_depths(zs, relay.z)
        self.times = _check_times(times)
        self.device = device or dev.require_cuda()
        cx = vg.x0 + (vg.nx // 2) * vg.dx
        cy = vg.y0 + (vg.ny // 2) * vg.dy
        rel = np.asarray(relay.points.points)
        nu_rx = (rel[:, 0] - cx) / vg.dx
        nu_ry = (rel[:, 1] - cy) / vg.dy
        lo_x, hi_x = -(vg.nx // 2), vg.nx - vg.nx // 2 - 1
        lo_y, hi_y = -(vg.ny // 2), vg.ny - vg.ny // 2 - 1
        lx = max(hi_x - nu_rx.min(), nu_rx.max() - lo_x)
        ly = max(hi_y - nu_ry.min(), nu_ry.max() - lo_y)
        on_lattice = (np.abs(nu_rx - np.round(nu_rx)).max() < 1e-9
                      and np.abs(nu_ry - np.round(nu_ry)).max() < 1e-9)
        # off-lattice points make the result depend on P: keep the reference rule
        # (SURVEY F3); lattice points are P-independent (F4), so pick a fast pad
        pad = _exact_pad if on_lattice else _pad_size
        px = pad(lx, max(abs(nu_rx).max(), vg.nx // 2), vg.nx)
        py = pad(ly, max(abs(nu_ry).max(), vg.ny // 2), vg.ny)
        self.px, self.py = px, py
        torus = np.column_stack([2.0 * np.pi * nu_rx / px, 2.0 * np.pi * nu_ry / py])
        self.plan = nu.NufftPlan((py, px), eps, self.device)
        self.pts = self.plan.points(torus)
        self.freqs = np.asarray(slices.frequencies, dtype=np.float64)
        self.n_illum = int(slices.illuminations.count)
        self._setup_prop(px, py, vg, relay.z, include_illumination,
                         plane_range or (0, vg.nz))
        F, I = self.freqs.size, self.n_illum
        self.uhat = torch.empty((F * I * py * px,), dtype=torch.complex64, device=self.device)
        self.fine = torch.empty((F * I, self.plan.fine_elems), dtype=torch.complex64,
                                device=self.device)
        self.ill = _ill_tensor(slices, self.device)
        self.frame_w = _frame_weights(self.freqs, self.times, self.device)
        self.n_frames = 1 if self.times is None else self.times.size
        self.grid = grid

    def relay_spectra(self, coeff, stream=None):
        F, I = self.freqs.size, self.n_illum
        nu.type1(self.plan, self.pts, coeff, F * I, coeff.shape[-1], self.uhat,
                 self.py * self.px, self.fine, self.prop.transposed, stream)
        return self.uhat

    def run(self, coeff, vol=None, stream=None):
        if vol is None:
            vol = torch.zeros((self.n_frames, self.n_voxels), dtype=torch.complex64,
                              device=self.device)
        else:
            vol.zero_()
        return self._propagate(self.relay_spectra(coeff, stream), vol, stream)


def nursd1(slices, grid, eps: float = 1e-6, times=None, threads: int = 1,
           include_illumination: bool = True):
    """Scattered planar relay -> cuboid via type-1 NUFFT (reconstruct.py:335-385)."""
    eng = cached_engine("nursd1", slices, grid, (float(eps), bool(include_illumination),
                                                 None if times is None else np.asarray(times)),
                        lambda: Nursd1Engine(slices, grid, eps, include_illumination, times))
    return _volume(grid, eng.run_dropin(device_coefficients(slices)), eng.times)


# ---------------------------------------------------------------------------
# type-2 readout family: nursd2, nursd3, srsd_nursd2 (reconstruct.py:393-586)
# ---------------------------------------------------------------------------


def _explicit_geo(grid, cx, cy, dx, dy, sx=1.0, sy=1.0):
    """Per-plane fractional lattice indices (reconstruct.py:393-410)."""
    geo, start = [], 0
    for pl in grid.planes:
        pts = np.asarray(pl.points.points)
        geo.append((start, pts.shape[0], sx * (pts[:, 0] - cx) / dx, sy * (pts[:, 1] - cy) / dy,
                    pts, float(pl.z)))
        start += pts.shape[0]
    return geo


_READOUT_BYTES = int(os.environ.get("PF_READOUT_MB", "256")) << 20   # spectra + fine grids per batch


class _Type2Readout:
    """cfft2(G_k) * Uhat -> nufft2 at the plane's voxels * scale * illumination phase."""

    def __init__(self, device, slices, grid, geo, px, py, lag_dx, lag_dy, z_src, eps,
                 include_illumination, times):
        self.device = device
        self.geo = geo
        self.px, self.py = px, py
        self.freqs = np.asarray(slices.frequencies, dtype=np.float64)
        self.n_illum = I = int(slices.illuminations.count)
        self.times = times
        self.n_frames = 1 if times is None else times.size
        self.count = grid.count
        self.include = bool(include_illumination)
        planes = [PlaneSpec(z - z_src, lag_dx, lag_dy, 0, 1, 0, 1, z, 0, i)
                  for i, (*_, z) in enumerate(geo)]
        self.plan = nu.NufftPlan((py, px), eps, device)
        # planes per launch: product spectra and fine grids of a whole batch resident
        per_plane = 8 * I * (self.plan.fine_elems + py * px)
        self.nb = max(1, min(len(planes), _READOUT_BYTES // per_plane))
        # readout over all frequencies in one launch per plane batch, on frequency-interleaved
        # fine grids (16 frequencies per group): ES window at w = 4, one illumination, static
        nf = self.freqs.size
        self.n_groups = -(-nf // 16)
        self.fused_f = bool(
            _READOUT_FUSED and self.plan.window == "es" and self.plan.w == 4 and I == 1
            and times is None and self.plan.fine_elems * 16 < (1 << 31)
            and _lib.call("pf_nufft_type2_il_ok", self.plan.gref))
        if self.fused_f:
            per_f = 8 * 16 * self.n_groups * self.plan.fine_elems
            self.nb = max(1, min(len(planes), self.nb, _READOUT_FUSED_BYTES // per_f))
        self.prop = Propagator(device, px, py, px, py, 0, 0, I, include_illumination, planes,
                               py * px, batch=self.nb)
        self.prop.geom.flags = 1      # register path off: generic product-only columns
        # every plane's points, cell-sorted within the plane, concatenated in plane order:
        # one interpolation launch serves a whole plane batch
        i0s, d0s, xyzs, pls, dsts, self.pt_lo = [], [], [], [], [], [0]
        psets = []
        for k, (start, cnt, nux, nuy, pts, z) in enumerate(geo):
            tor = np.column_stack([2.0 * np.pi * nux / px, 2.0 * np.pi * nuy / py])
            npts = self.plan.points(tor, cell_sorted=True)
            psets.append(npts)
            xyz = np.column_stack([pts[:, 0], pts[:, 1], np.full(cnt, z)])[npts.order]
            i0s.append(npts.i0)
            d0s.append(npts.d0)
            xyzs.append(xyz)
            pls.append(np.full(cnt, k, dtype=np.int32))
            dsts.append(start + npts.order.astype(np.int64))
            self.pt_lo.append(self.pt_lo[-1] + cnt)
        # the fine cells any voxel's stencil touches: the type-2 start forms no others
        self.window = nu.stencil_window(self.plan, psets) if _T2_WINDOW else None
        self.i0_all = torch.cat(i0s)
        self.d0_all = torch.cat(d0s)
        self.xyz_all = torch.from_numpy(np.ascontiguousarray(np.vstack(xyzs))).to(device)
        self.plane_all = torch.from_numpy(np.concatenate(pls)).to(device)
        self.dst_all = torch.from_numpy(np.concatenate(dsts)).to(device)
        self.n_planes = len(geo)
        self.spec = torch.empty((self.nb * I * py * px,), dtype=torch.complex64, device=device)
        self.fine = torch.empty((self.nb * I, self.plan.fine_elems), dtype=torch.complex64,
                                device=device)
        self.ill = _ill_tensor(slices, device)
        self.frame_w = _frame_weights(self.freqs, times, device)
        if self.fused_f:
            # zero once: the slots of frequencies beyond F and the cells outside the stencil
            # window are never written, the rest is rewritten every run
            self.fine_f = torch.zeros((self.n_groups * self.nb * self.plan.fine_elems * 16,),
                                      dtype=torch.complex64, device=device)
            self.kturns = torch.from_numpy(self.freqs / (C * 2.0 * np.pi)).to(device)

    def _run_fused(self, uhat_of, vol, stream):
        """Per plane batch: every frequency's product spectra and type-2 start into the
        frequency-interleaved fine grids, then one readout launch over all frequencies."""
        s = dev.stream_ptr(stream)
        py, px, p = self.py, self.px, self.plan
        gref = ctypes.byref(self.prop.geom)
        base = dev.ptr(self.prop.planes_dev)
        fe = p.fine_elems
        c0, nc, r0, nr = self.window or (0, p.mrs[2], 0, p.mrs[1])
        gstride = self.nb * fe * 16
        for b0 in range(0, self.n_planes, self.nb):
            n = min(self.nb, self.n_planes - b0)
            pp = base + b0 * self.prop.plane_size
            for fi in range(self.freqs.size):
                khat = float(self.freqs[fi]) / C
                _lib.call("pf_prop_kernel_rows", pp, n, khat, gref, self.prop.plan_x.ref,
                          dev.ptr(self.prop.ws_a), s)
                _lib.call("pf_prop_columns", pp, n, gref, self.prop.plan_y.ref,
                          dev.ptr(self.prop.ws_a), dev.ptr(uhat_of(fi)), dev.ptr(self.spec), 1, s)
                _lib.call("pf_nufft_type2_start_2d_ilm", p.gref, dev.ptr(self.spec), py * px,
                          dev.ptr(p.kers[1]), dev.ptr(p.kers[2]), n, dev.ptr(self.fine), fe,
                          dev.fft_plan(p.mrs[2], p.device).ref, dev.fft_plan(p.mrs[1], p.device).ref,
                          c0, nc, r0, nr, dev.ptr(self.fine_f) + 8 * (fi // 16) * gstride, 16,
                          fi % 16, s)
            lo, hi = self.pt_lo[b0], self.pt_lo[b0 + n]
            if hi > lo:
                _lib.call("pf_nufft_interp2_freqs", p.gref, dev.ptr(self.i0_all) + 12 * lo,
                          dev.ptr(self.d0_all) + 12 * lo, dev.ptr(self.xyz_all) + 24 * lo,
                          dev.ptr(self.plane_all) + 4 * lo, dev.ptr(self.dst_all) + 8 * lo,
                          hi - lo, b0, dev.ptr(self.fine_f), fe * 16, gstride, self.freqs.size,
                          dev.ptr(self.kturns), dev.ptr(self.ill), int(self.include),
                          1.0 / (px * py), dev.ptr(self.frame_w), dev.ptr(vol), s)
        return vol

    def run(self, uhat_of, vol, stream=None):
        if self.fused_f:
            return self._run_fused(uhat_of, vol, stream)
        s = dev.stream_ptr(stream)
        I, py, px = self.n_illum, self.py, self.px
        gref = ctypes.byref(self.prop.geom)
        base = dev.ptr(self.prop.planes_dev)
        nplanes = self.n_planes
        for fi in range(self.freqs.size):
            khat = float(self.freqs[fi]) / C
            uhat = uhat_of(fi)
            fw = dev.ptr(self.frame_w) + 8 * fi * self.n_frames
            for b0 in range(0, nplanes, self.nb):
                n = min(self.nb, nplanes - b0)
                pp = base + b0 * self.prop.plane_size
                _lib.call("pf_prop_kernel_rows", pp, n, khat, gref, self.prop.plan_x.ref,
                          dev.ptr(self.prop.ws_a), s)
                _lib.call("pf_prop_columns", pp, n, gref, self.prop.plan_y.ref,
                          dev.ptr(self.prop.ws_a), dev.ptr(uhat), dev.ptr(self.spec), 1, s)
                nu.place_and_inverse(self.plan, self.spec, n * I, py * px, self.fine, stream,
                                     self.window)
                lo, hi = self.pt_lo[b0], self.pt_lo[b0 + n]
                fe = self.plan.fine_elems
                _lib.call("pf_nufft_interp2_batch", self.plan.gref,
                          dev.ptr(self.i0_all) + 12 * lo, dev.ptr(self.d0_all) + 12 * lo,
                          dev.ptr(self.xyz_all) + 24 * lo, dev.ptr(self.plane_all) + 4 * lo,
                          dev.ptr(self.dst_all) + 8 * lo, hi - lo, b0, dev.ptr(self.fine),
                          I * fe, fe, I, dev.ptr(self.ill), khat, int(self.include),
                          1.0 / (px * py), fw, self.n_frames, dev.ptr(vol), self.count, s)
        return vol


# ---------------------------------------------------------------------------
# arbitrary voxel depths: z-Chebyshev type-2 readout
# ---------------------------------------------------------------------------

_READOUT_FUSED = os.environ.get("PF_READOUT_FUSED", "1") != "0"   # all frequencies per readout launch
_READOUT_FUSED_BYTES = int(os.environ.get("PF_READOUT_FUSED_MB", "2048")) << 20
_T2_WINDOW = os.environ.get("PF_T2_WINDOW", "1") != "0"   # type-2 start limited to the stencils' cells
_ZCHEB_IL = os.environ.get("PF_ZCHEB_IL", "1") != "0"      # node-interleaved fine grids in the readout
_ZCHEB_NODES = int(os.environ.get("PF_ZCHEB_NODES", "12"))
_ZCHEB_KAPPA = float(os.environ.get("PF_ZCHEB_KAPPA", "6.0"))   # k_max x slab thickness


def zcheb_slabs(zs, k_max: float, nodes: int = _ZCHEB_NODES, kappa: float = _ZCHEB_KAPPA):
    """Depth slabs and Chebyshev nodes for voxels at depths ``zs``.

    Across a slab of thickness dz the kernel spectrum Ghat_z(k) of the reference's
    nursd2 (the DFT of exp(i k r)/r sampled on the pad, reconstruct.py:128-130,443) turns
    by at most k dz in phase; with k_max dz = kappa and n Chebyshev nodes per slab the
    interpolation of exp(i k_max z) is accurate to 2.6e-7 at kappa = 6, n = 12 (4.4e-7 at
    4 / 10, 3.9e-6 at 3 / 8; measured on 50,000 random depths).  Returns
    (edges [S + 1], nodes [S, n], slab index per voxel, Lagrange weights [N, n])."""
    zs = np.asarray(zs, dtype=np.float64)
    z0, z1 = float(zs.min()), float(zs.max())
    span = max(z1 - z0, 1e-12)
    S = max(1, math.ceil(k_max * span / kappa))
    edges = z0 + span * np.arange(S + 1) / S
    mid, half = 0.5 * (edges[1:] + edges[:-1]), 0.5 * (edges[1:] - edges[:-1])
    j = np.arange(nodes)
    theta = np.pi * (2 * j + 1) / (2 * nodes)
    xn = np.cos(theta)                                   # Chebyshev points of the first kind
    node_z = mid[:, None] + half[:, None] * xn[None, :]
    slab = np.minimum(S - 1, np.floor((zs - z0) / span * S).astype(np.int64))
    x = (zs - mid[slab]) / half[slab]
    # barycentric Lagrange weights for first-kind Chebyshev points (float64)
    bw = ((-1.0) ** j) * np.sin(theta)
    diff = x[:, None] - xn[None, :]
    exact = np.abs(diff) < 1e-15
    diff[exact] = 1.0
    t = bw[None, :] / diff
    lw = t / t.sum(axis=1, keepdims=True)
    rows = exact.any(axis=1)
    if rows.any():
        lw[rows] = exact[rows].astype(np.float64)
    return edges, node_z, slab, lw


class _ZChebReadout:
    """nursd2 at voxels of arbitrary depth: the kernel spectra are formed at the Chebyshev
    nodes of depth slabs (product spectra Uhat * Ghat_node, place + inverse fine-grid FFT
    per node, as the plane readout does per plane), and each voxel's value is the
    Lagrange-weighted sum over its slab's nodes of the same type-2 stencil
    (``pf_nufft_interp2_nodes``), times its own illumination phase at its exact depth
    (reconstruct.py:455).  Equals nursd2 on one plane per voxel up to the interpolation
    error of Ghat_z in z (``zcheb_slabs``)."""

    def __init__(self, device, slices, points, cx, cy, dx, dy, px, py, z_src, eps,
                 include_illumination, times):
        self.device = device
        self.px, self.py = px, py
        self.freqs = np.asarray(slices.frequencies, dtype=np.float64)
        self.n_illum = I = int(slices.illuminations.count)
        self.times = times
        self.n_frames = 1 if times is None else times.size
        pts = np.asarray(points, dtype=np.float64)
        self.count = pts.shape[0]
        self.include = bool(include_illumination)
        k_max = float(self.freqs.max()) / C
        edges, node_z, slab, lw = zcheb_slabs(pts[:, 2], k_max)
        S, M = node_z.shape
        self.n_slabs, self.nodes = S, M
        planes = [PlaneSpec(float(z) - z_src, dx, dy, 0, 1, 0, 1, float(z), 0, i)
                  for i, z in enumerate(node_z.ravel())]
        self.plan = nu.NufftPlan((py, px), eps, device)
        per_plane = 8 * I * (self.plan.fine_elems + py * px)
        self.slabs_per_batch = max(1, min(S, _READOUT_BYTES // (M * per_plane)))
        self.nb = self.slabs_per_batch * M
        self.prop = Propagator(device, px, py, px, py, 0, 0, I, include_illumination, planes,
                               py * px, batch=self.nb)
        self.prop.geom.flags = 1      # generic product-only columns
        # voxels slab by slab, cell-sorted within a slab; each carries its slab's first
        # node plane and its node weights
        i0s, d0s, xyzs, pls, dsts, lws, self.pt_lo = [], [], [], [], [], [], [0]
        psets = []
        for s in range(S):
            idx = np.nonzero(slab == s)[0]
            if idx.size:
                sp = pts[idx]
                tor = np.column_stack([2.0 * np.pi * (sp[:, 0] - cx) / dx / px,
                                       2.0 * np.pi * (sp[:, 1] - cy) / dy / py])
                npts = self.plan.points(tor, cell_sorted=True)
                psets.append(npts)
                o = npts.order
                i0s.append(npts.i0)
                d0s.append(npts.d0)
                xyzs.append(sp[o])
                pls.append(np.full(idx.size, s * M, dtype=np.int32))
                dsts.append(idx[o].astype(np.int64))
                lws.append(lw[idx[o]])
            self.pt_lo.append(self.pt_lo[-1] + idx.size)
        self.window = nu.stencil_window(self.plan, psets) if _T2_WINDOW else None
        cat = torch.cat
        self.i0_all = cat(i0s)
        self.d0_all = cat(d0s)
        self.xyz_all = torch.from_numpy(np.ascontiguousarray(np.vstack(xyzs))).to(device)
        self.plane_all = torch.from_numpy(np.concatenate(pls)).to(device)
        self.dst_all = torch.from_numpy(np.concatenate(dsts)).to(device)
        self.lw_all = torch.from_numpy(np.ascontiguousarray(np.vstack(lws)).astype(np.float32)).to(device)
        self.spec = torch.empty((self.nb * I * py * px,), dtype=torch.complex64, device=device)
        self.fine = torch.empty((self.nb * I, self.plan.fine_elems), dtype=torch.complex64,
                                device=device)
        self.ill = _ill_tensor(slices, device)
        self.frame_w = _frame_weights(self.freqs, times, device)
        # node-interleaved fine grids (a tap's node values contiguous: wide loads in the
        # readout): ES window at w = 4, 12 nodes, one illumination, split column pass
        self.interleaved = bool(
            _ZCHEB_IL and self.plan.window == "es" and self.plan.w == 4 and M == 12 and I == 1
            and self.plan.fine_elems * M < (1 << 31)
            and _lib.call("pf_nufft_type2_il_ok", self.plan.gref))
        self.fine_il = torch.empty_like(self.fine) if self.interleaved else None

    def run(self, uhat_of, vol, stream=None):
        s = dev.stream_ptr(stream)
        I, py, px, M = self.n_illum, self.py, self.px, self.nodes
        gref = ctypes.byref(self.prop.geom)
        base = dev.ptr(self.prop.planes_dev)
        fe = self.plan.fine_elems
        for fi in range(self.freqs.size):
            khat = float(self.freqs[fi]) / C
            uhat = uhat_of(fi)
            fw = dev.ptr(self.frame_w) + 8 * fi * self.n_frames
            for s0 in range(0, self.n_slabs, self.slabs_per_batch):
                s1 = min(self.n_slabs, s0 + self.slabs_per_batch)
                b0, n = s0 * M, (s1 - s0) * M
                pp = base + b0 * self.prop.plane_size
                _lib.call("pf_prop_kernel_rows", pp, n, khat, gref, self.prop.plan_x.ref,
                          dev.ptr(self.prop.ws_a), s)
                _lib.call("pf_prop_columns", pp, n, gref, self.prop.plan_y.ref,
                          dev.ptr(self.prop.ws_a), dev.ptr(uhat), dev.ptr(self.spec), 1, s)
                lo, hi = self.pt_lo[s0], self.pt_lo[s1]
                if self.interleaved:
                    p = self.plan
                    c0, nc, r0, nr = self.window or (0, p.mrs[2], 0, p.mrs[1])
                    _lib.call("pf_nufft_type2_start_2d_il", p.gref, dev.ptr(self.spec), py * px,
                              dev.ptr(p.kers[1]), dev.ptr(p.kers[2]), n, dev.ptr(self.fine), fe,
                              dev.fft_plan(p.mrs[2], p.device).ref,
                              dev.fft_plan(p.mrs[1], p.device).ref, c0, nc, r0, nr,
                              dev.ptr(self.fine_il), M, s)
                    if hi > lo:
                        _lib.call("pf_nufft_interp2_nodes_il", p.gref,
                                  dev.ptr(self.i0_all) + 12 * lo, dev.ptr(self.d0_all) + 12 * lo,
                                  dev.ptr(self.xyz_all) + 24 * lo, dev.ptr(self.plane_all) + 4 * lo,
                                  dev.ptr(self.dst_all) + 8 * lo, hi - lo, b0,
                                  dev.ptr(self.fine_il), fe * M, dev.ptr(self.ill), khat,
                                  int(self.include), 1.0 / (px * py), fw, self.n_frames,
                                  dev.ptr(vol), self.count, M, dev.ptr(self.lw_all) + 4 * M * lo, s)
                    continue
                nu.place_and_inverse(self.plan, self.spec, n * I, py * px, self.fine, stream,
                                     self.window)
                if hi == lo:
                    continue
                _lib.call("pf_nufft_interp2_nodes", self.plan.gref,
                          dev.ptr(self.i0_all) + 12 * lo, dev.ptr(self.d0_all) + 12 * lo,
                          dev.ptr(self.xyz_all) + 24 * lo, dev.ptr(self.plane_all) + 4 * lo,
                          dev.ptr(self.dst_all) + 8 * lo, hi - lo, b0, dev.ptr(self.fine),
                          I * fe, fe, I, dev.ptr(self.ill), khat, int(self.include),
                          1.0 / (px * py), fw, self.n_frames, dev.ptr(vol), self.count, M,
                          dev.ptr(self.lw_all) + 4 * M * lo, s)
        return vol


class Nursd2VoxelsEngine(GraphedRun):
    """nursd2 (reconstruct.py:413-459) onto voxels at arbitrary depths (``VoxelCloud``):
    the reference's pads and spectra, the z-Chebyshev readout (:class:`_ZChebReadout`)."""

    def __init__(self, slices, cloud, eps: float = 1e-6, times=None,
                 include_illumination: bool = True, device=None):
        _require(_kind(cloud) == "voxels", "this algorithm reconstructs onto a voxel cloud")
        relay = _uniform_relay(slices)
        g = relay.grid
        cx, cy = g.center()
        pts = np.asarray(cloud.points, dtype=np.float64)
        _check_depths(pts[:, 2], g.z)
        self.times = _check_times(times)
        self.device = device or dev.require_cuda()
        jx_lo, jx_hi = -(g.nx // 2), g.nx - g.nx // 2 - 1
        jy_lo, jy_hi = -(g.ny // 2), g.ny - g.ny // 2 - 1
        ax = (pts[:, 0] - cx) / g.dx
        ay = (pts[:, 1] - cy) / g.dy
        px = _pad_size(max(ax.max() - jx_lo, jx_hi - ax.min()), max(abs(ax).max(), g.nx // 2),
                       g.nx)
        py = _pad_size(max(ay.max() - jy_lo, jy_hi - ay.min()), max(abs(ay).max(), g.ny // 2),
                       g.ny)
        self.relay_grid, self.px, self.py = g, px, py
        self.ro = _ZChebReadout(self.device, slices, pts, cx, cy, g.dx, g.dy, px, py, g.z, eps,
                                include_illumination, self.times)
        self.freqs, self.n_illum, self.n_frames = self.ro.freqs, self.ro.n_illum, self.ro.n_frames
        self.n_voxels = cloud.count
        F, I = self.freqs.size, self.n_illum
        self.uhat = torch.empty((F * I * py * px,), dtype=torch.complex64, device=self.device)

    def run(self, coeff, vol=None, stream=None):
        if vol is None:
            vol = torch.zeros((self.n_frames, self.n_voxels), dtype=torch.complex64,
                              device=self.device)
        else:
            vol.zero_()
        uhat = self.relay_spectra(coeff, stream)
        per_f = self.n_illum * self.py * self.px
        return self.ro.run(lambda fi: uhat[fi * per_f:], vol, stream)


def nursd2_voxels(slices, cloud, eps: float = 1e-6, times=None, threads: int = 1,
                  include_illumination: bool = True):
    """Uniform relay -> voxels at arbitrary (x, y, z) (``VoxelCloud``): nursd2 semantics
    (reconstruct.py:413-459 on one plane per voxel) by the z-Chebyshev readout."""
    eng = Nursd2VoxelsEngine(slices, cloud, eps, times, include_illumination)
    return _volume(cloud, eng.run(device_coefficients(slices)), eng.times)


def _readout_setup(slices, grid, times):
    _require(_kind(grid) == "explicit", "this algorithm reconstructs onto explicit voxels")
    return dev.require_cuda(), _check_times(times)


class Nursd2Engine(GraphedRun):
    """Device plan of :func:`nursd2` (reconstruct.py:413-459) for one geometry; reusable.

    ``slices`` only supplies geometry (uniform relay, frequencies, illuminations);
    ``run(coeff)`` takes frequency-major device coefficients [F, I, D].
    """

    def __init__(self, slices, grid, eps: float = 1e-6, times=None,
                 include_illumination: bool = True, device=None):
        _require(_kind(grid) == "explicit", "nursd2 reconstructs onto explicit voxels")
        relay = _uniform_relay(slices)
        g = relay.grid
        cx, cy = g.center()
        geo = _explicit_geo(grid, cx, cy, g.dx, g.dy)
        _check_depths(np.asarray([t[-1] for t in geo]), g.z)
        self.times = _check_times(times)
        self.device = device or dev.require_cuda()
        jx_lo, jx_hi = -(g.nx // 2), g.nx - g.nx // 2 - 1
        jy_lo, jy_hi = -(g.ny // 2), g.ny - g.ny // 2 - 1
        ax = np.concatenate([t[2] for t in geo])
        ay = np.concatenate([t[3] for t in geo])
        px = _pad_size(max(ax.max() - jx_lo, jx_hi - ax.min()), max(abs(ax).max(), g.nx // 2),
                       g.nx)
        py = _pad_size(max(ay.max() - jy_lo, jy_hi - ay.min()), max(abs(ay).max(), g.ny // 2),
                       g.ny)
        self.relay_grid, self.px, self.py = g, px, py
        self.ro = _Type2Readout(self.device, slices, grid, geo, px, py, g.dx, g.dy, g.z, eps,
                                include_illumination, self.times)
        self.freqs, self.n_illum, self.n_frames = self.ro.freqs, self.ro.n_illum, self.ro.n_frames
        self.n_voxels = grid.count
        F, I = self.freqs.size, self.n_illum
        self.uhat = torch.empty((F * I * py * px,), dtype=torch.complex64, device=self.device)

    def relay_spectra(self, coeff, stream=None):
        """Uhat_f = cfft2(pad_embed(u_f)), natural order (reconstruct.py:441-443)."""
        g, F, I = self.relay_grid, self.freqs.size, self.n_illum
        _lib.call("pf_embed_centered", dev.ptr(coeff), F * I, g.ny, g.nx, g.ny * g.nx,
                  dev.ptr(self.uhat), self.py, self.px, 0, dev.stream_ptr(stream))
        dev.fft2_natural(self.uhat, self.py, self.px, F * I, -1, 1.0, stream)
        return self.uhat

    def run(self, coeff, vol=None, stream=None):
        if vol is None:
            vol = torch.zeros((self.n_frames, self.n_voxels), dtype=torch.complex64,
                              device=self.device)
        else:
            vol.zero_()
        uhat = self.relay_spectra(coeff, stream)
        per_f = self.n_illum * self.py * self.px
        return self.ro.run(lambda fi: uhat[fi * per_f:], vol, stream)


Nursd2VoxelsEngine.relay_spectra = Nursd2Engine.relay_spectra   # same spectra (reconstruct.py:441-443)


def nursd2(slices, grid, eps: float = 1e-6, times=None, threads: int = 1,
           include_illumination: bool = True):
    """Uniform relay -> explicit voxels (reconstruct.py:413-459)."""
    eng = Nursd2Engine(slices, grid, eps, times, include_illumination)
    return _volume(grid, eng.run(device_coefficients(slices)), eng.times)


def nursd3(slices, grid, eps: float = 1e-6, lattice_pitch: float | None = None, times=None,
           threads: int = 1, include_illumination: bool = True):
    """Scattered planar relay -> explicit voxels through a virtual lattice (reconstruct.py:467-525)."""
    _require(_kind(grid) == "explicit", "nursd3 reconstructs onto explicit voxels")
    relay = _planar_relay(slices)
    pitch = (float(lattice_pitch) if lattice_pitch is not None
             else slices.shortest_wavelength / 2.0)
    _require(pitch > 0, "lattice pitch must be > 0")
    rel = np.asarray(relay.points.points)
    tgt = np.vstack([np.asarray(p.points.points) for p in grid.planes])
    lo = np.minimum(rel.min(axis=0), tgt.min(axis=0))
    hi = np.maximum(rel.max(axis=0), tgt.max(axis=0))
    anchor = rel[0] + np.round(((lo + hi) / 2.0 - rel[0]) / pitch) * pitch
    cx, cy = float(anchor[0]), float(anchor[1])
    nu_rx = (rel[:, 0] - cx) / pitch
    nu_ry = (rel[:, 1] - cy) / pitch
    geo = _explicit_geo(grid, cx, cy, pitch, pitch)
    _check_depths(np.asarray([t[-1] for t in geo]), relay.z)
    times = _check_times(times)
    device = dev.require_cuda()
    ax = np.concatenate([t[2] for t in geo])
    ay = np.concatenate([t[3] for t in geo])
    px = _pad_size(max(ax.max() - nu_rx.min(), nu_rx.max() - ax.min()),
                   max(abs(ax).max(), abs(nu_rx).max()), 1)
    py = _pad_size(max(ay.max() - nu_ry.min(), nu_ry.max() - ay.min()),
                   max(abs(ay).max(), abs(nu_ry).max()), 1)
    ro = _Type2Readout(device, slices, grid, geo, px, py, pitch, pitch, float(relay.z), eps,
                       include_illumination, times)
    coeff = device_coefficients(slices)
    F, I = ro.freqs.size, ro.n_illum
    plan = nu.NufftPlan((py, px), eps, device)
    pts = plan.points(np.column_stack([2.0 * np.pi * nu_rx / px, 2.0 * np.pi * nu_ry / py]))
    uhat = torch.empty((F * I * py * px,), dtype=torch.complex64, device=device)
    nu.type1(plan, pts, coeff, F * I, coeff.shape[-1], uhat, py * px)
    vol = torch.zeros((ro.n_frames, grid.count), dtype=torch.complex64, device=device)
    ro.run(lambda fi: uhat[fi * I * py * px:], vol)
    return _volume(grid, vol, times)


def srsd_nursd2(slices, grid, alpha: float, beta: float | None = None, eps: float = 1e-6,
                times=None, threads: int = 1, include_illumination: bool = True):
    """Uniform relay -> explicit voxels through one scaled transform (reconstruct.py:533-586)."""
    _require(_kind(grid) == "explicit", "srsd-nursd2 reconstructs onto explicit voxels")
    if beta is None:
        beta = alpha
    _require(0 < alpha <= 1 and 0 < beta <= 1, "scale factors must lie in (0, 1]")
    relay = _uniform_relay(slices)
    g = relay.grid
    cx, cy = g.center()
    geo = _explicit_geo(grid, cx, cy, g.dx, g.dy, alpha, beta)
    _check_depths(np.asarray([t[-1] for t in geo]), g.z)
    times = _check_times(times)
    device = dev.require_cuda()
    jx_lo, jx_hi = -(g.nx // 2), g.nx - g.nx // 2 - 1
    jy_lo, jy_hi = -(g.ny // 2), g.ny - g.ny // 2 - 1
    ax = np.concatenate([t[2] for t in geo])
    ay = np.concatenate([t[3] for t in geo])
    px = _pad_size(max(ax.max() - alpha * jx_lo, alpha * jx_hi - ax.min()),
                   max(abs(ax).max(), g.nx // 2), g.nx)
    py = _pad_size(max(ay.max() - beta * jy_lo, beta * jy_hi - ay.min()),
                   max(abs(ay).max(), g.ny // 2), g.ny)
    ro = _Type2Readout(device, slices, grid, geo, px, py, g.dx / alpha, g.dy / beta, g.z, eps,
                       include_illumination, times)
    coeff = device_coefficients(slices)
    F, I = ro.freqs.size, ro.n_illum
    tabs = _ScaledTables(px, py, [alpha], [beta], device)
    uhat = torch.empty((F * I * py * px,), dtype=torch.complex64, device=device)
    xbuf = torch.empty((g.ny * px,), dtype=torch.complex64, device=device)
    for fi in range(F):
        for p in range(I):
            _scaled_spectra(coeff[fi, p], g.ny, g.nx, py, px, tabs, 0, 1, xbuf,
                            uhat[(fi * I + p) * py * px:], py * px, False)
    vol = torch.zeros((ro.n_frames, grid.count), dtype=torch.complex64, device=device)
    ro.run(lambda fi: uhat[fi * I * py * px:], vol)
    return _volume(grid, vol, times)


# ---------------------------------------------------------------------------
# nursd3d: scattered 3D relay -> cuboid (reconstruct.py:594-765)
# ---------------------------------------------------------------------------


class _FlatSlices:
    """A 3D relay whose points share one z viewed as a planar relay (reconstruct.py:735-740)."""

    def __init__(self, slices, rel):
        from .core import NonUniformPlanarRelay, PointList
        self.frequencies = slices.frequencies
        self.illuminations = slices.illuminations
        self.relay = NonUniformPlanarRelay(PointList(rel[:, :2]), float(rel[0, 2]))
        self._src = slices
        self.n_freq = int(np.asarray(slices.frequencies).size)

    @property
    def coefficients(self):
        return self._src.coefficients

    @property
    def device_coefficients(self):
        return device_coefficients(self._src)


def _lattice_3d(slices, grid, z_pitch):
    """Virtual-lattice geometry shared by the non-planar algorithms (reconstruct.py:594-621)."""
    relay = _nonplanar_relay(slices)
    vg = grid.grid
    rel = np.asarray(relay.points.points)
    dz3 = float(z_pitch) if z_pitch else slices.shortest_wavelength / 2.0
    _require(dz3 > 0, "depth lattice pitch must be > 0")
    z_min = float(rel[:, 2].min())
    z_ext = float(rel[:, 2].max()) - z_min
    nz3 = max(1, math.ceil(z_ext / dz3) + 1)
    pz = next_fast_len(2 * nz3 + 2)
    z0 = z_min + nz3 * dz3
    zs = vg.z_coords()
    _require(bool((zs > z0).all()),
             "every voxel plane must lie beyond the relay surface's far face "
             f"(z > {z0:.6g})")
    cx = vg.x0 + (vg.nx // 2) * vg.dx
    cy = vg.y0 + (vg.ny // 2) * vg.dy
    nu_rx = (rel[:, 0] - cx) / vg.dx
    nu_ry = (rel[:, 1] - cy) / vg.dy
    lo_x, hi_x = -(vg.nx // 2), vg.nx - vg.nx // 2 - 1
    lo_y, hi_y = -(vg.ny // 2), vg.ny - vg.ny // 2 - 1
    lx = max(hi_x - nu_rx.min(), nu_rx.max() - lo_x)
    ly = max(hi_y - nu_ry.min(), nu_ry.max() - lo_y)
    px = _pad_size(lx, max(abs(nu_rx).max(), vg.nx // 2), vg.nx)
    py = _pad_size(ly, max(abs(nu_ry).max(), vg.ny // 2), vg.ny)
    slab = pz // 2 + (nz3 - nz3 // 2)
    return rel, dz3, z_min, nz3, pz, z0, nu_rx, nu_ry, px, py, slab


_GROUP_FINE_BYTES = 4 << 30   # type-1 fine grids of one nursd3d frequency group
_G3_EVEN = os.environ.get("PF_G3_EVEN", "1") != "0"   # 3D kernel transform on the even octant


class _Lattice3dEngine(_UhatPropEngine):
    """Shared two-stage structure of nursd3d / rsd3d (reconstruct.py:662-765): stage 1
    forms the virtual-lattice spectrum (subclass), x cfft_n(G3) -> cifft_n -> slab ->
    cfft_2d; stage 2 propagates the virtual plane to every output plane."""

    def _setup_lattice(self, slices, grid, z_pitch, include_illumination, times, device,
                       plane_range):
        _require(_kind(grid) == "cuboid", self.GRID_MSG)
        geo = _lattice_3d(slices, grid, z_pitch)
        (rel, dz3, z_min, nz3, pz, z0, nu_rx, nu_ry, px, py, slab) = geo
        self.times = _check_times(times)
        self.device = device or dev.require_cuda()
        vg = grid.grid
        self.vg, self.grid = vg, grid
        self.px, self.py, self.pz, self.dz3, self.z0 = px, py, pz, dz3, z0
        self.slab_nat = (slab - pz // 2) % pz
        zw = np.exp(2j * np.pi * ((np.arange(pz) * self.slab_nat) % pz) / pz)   # float64 phases
        self._zslab_w = torch.from_numpy(zw.astype(np.complex64)).to(self.device)
        self.freqs = np.asarray(slices.frequencies, dtype=np.float64)
        self.n_illum = int(slices.illuminations.count)
        self._setup_prop(px, py, vg, z0, include_illumination, plane_range or (0, vg.nz))
        self.ill = _ill_tensor(slices, self.device)
        self.frame_w = _frame_weights(self.freqs, self.times, self.device)
        self.n_frames = 1 if self.times is None else self.times.size
        return geo

    def virtual_planes(self, coeff, stream=None):
        """wave[slab] per (f, illumination), natural order [F*I][py][px] (reconstruct.py:741-760)."""
        F, I = self.freqs.size, self.n_illum
        px, py, pz = self.px, self.py, self.pz
        n3 = pz * py * px
        s = dev.stream_ptr(stream)
        gf = max(1, min(F, getattr(self, "group_f", 1)))   # frequencies per lattice-spectrum call
        uhat3g = torch.empty((gf * I * n3,), dtype=torch.complex64, device=self.device)
        g3g = torch.empty((gf * n3,), dtype=torch.complex64, device=self.device)
        out = torch.empty((F * I * py * px,), dtype=torch.complex64, device=self.device)
        for f0 in range(0, F, gf):
            f1 = min(F, f0 + gf)
            ng = f1 - f0
            self._lattice_spectra(coeff, f0, f1, uhat3g, n3, stream)
            # the group's kernels, then every later step once for the whole group (one launch
            # per pass over ng frequencies instead of ng small ones)
            for j, fi in enumerate(range(f0, f1)):
                _lib.call("pf_kernel3d", dev.ptr(g3g) + 8 * j * n3, pz, py, px, self.vg.dx,
                          self.vg.dy, self.dz3, float(self.freqs[fi]) / C, s)
            if _G3_EVEN and min(pz, py, px) >= 2:
                # G3 is even in every lag, so is its transform: each pass runs only over the
                # non-negative half of the other two axes (a quarter of the lines), the
                # mirrored half of the pass' own axis is filled by copy, and the product
                # reads the spectrum folded onto its octant
                hz, hy, hx = pz // 2, py // 2, px // 2
                g3p = dev.ptr(g3g)
                _lib.call("pf_fft_lines3", g3p, dev.fft_plan(px, self.device).ref,
                          ng * (hz + 1) * (hy + 1), hy + 1, px, hz + 1, py * px, n3, 1, -1, 1.0, s)
                _lib.call("pf_mirror_fill", g3p, ng, pz, py, px, 1, hz, hx, s)
                _lib.call("pf_fft_lines3", g3p, dev.fft_plan(py, self.device).ref,
                          ng * (hz + 1) * (hx + 1), hx + 1, 1, hz + 1, py * px, n3, px, -1, 1.0, s)
                _lib.call("pf_mirror_fill", g3p, ng, pz, py, px, 0, hy, hx, s)
                _lib.call("pf_fft_lines3", g3p, dev.fft_plan(pz, self.device).ref,
                          ng * (hy + 1) * (hx + 1), hx + 1, 1, hy + 1, px, n3, py * px, -1, 1.0, s)
                _lib.call("pf_cmul_even", dev.ptr(uhat3g), g3p, ng, I, pz, py, px, 1.0, s)
            else:
                dev.fftn_natural(g3g, (pz, py, px), ng, -1, 1.0, stream)
                if I == 1:
                    _lib.call("pf_cmul", dev.ptr(uhat3g), dev.ptr(g3g), ng * n3, ng * n3, 1.0, s)
                else:
                    for j in range(ng):
                        _lib.call("pf_cmul", dev.ptr(uhat3g) + 8 * j * I * n3,
                                  dev.ptr(g3g) + 8 * j * n3, I * n3, n3, 1.0, s)
            # cifft_n, then the slab plane: the z pass is evaluated at the slab only, then
            # the plane's y/x inverse transforms (the 3D inverse is never formed)
            out_g = out[f0 * I * py * px:f1 * I * py * px]
            _lib.call("pf_zslab", dev.ptr(uhat3g), ng * I, pz, py * px, dev.ptr(self._zslab_w),
                      1.0 / n3, dev.ptr(out_g), s)
            dev.fft2_natural(out_g, py, px, ng * I, +1, 1.0, stream)
        return out

    def _lattice_spectra(self, coeff, f0, f1, uhat3g, n3, stream):
        """Lattice spectra of frequencies [f0, f1) into uhat3g ([f][I][n3]); one call per
        frequency unless the subclass batches them."""
        I = self.n_illum
        for j, fi in enumerate(range(f0, f1)):
            self._lattice_spectrum(coeff[fi], uhat3g[j * I * n3:(j + 1) * I * n3], n3, stream)

    def relay_spectra(self, coeff, stream=None):
        F, I = self.freqs.size, self.n_illum
        px, py = self.px, self.py
        out = self.virtual_planes(coeff, stream)
        if self.prop.transposed:
            t = out.view(F * I, py, px).transpose(1, 2).contiguous()
            dev.fft2_natural(t, px, py, F * I, -1, 1.0, stream)
            return t.view(-1)
        dev.fft2_natural(out, py, px, F * I, -1, 1.0, stream)
        return out

    def run(self, coeff, vol=None, stream=None):
        if vol is None:
            vol = torch.zeros((self.n_frames, self.n_voxels), dtype=torch.complex64,
                              device=self.device)
        else:
            vol.zero_()
        return self._propagate(self.relay_spectra(coeff, stream), vol, stream)


class Nursd3dEngine(_Lattice3dEngine):
    """Stage 1 by a 3D type-1 NUFFT of the scattered relay (reconstruct.py:741-760)."""

    GRID_MSG = "nursd3d reconstructs onto a cuboid grid"

    def __init__(self, slices, grid, eps=1e-6, z_pitch=None, include_illumination=True,
                 times=None, device=None, plane_range=None):
        (rel, dz3, z_min, nz3, pz, z0, nu_rx, nu_ry, px, py, slab) = self._setup_lattice(
            slices, grid, z_pitch, include_illumination, times, device, plane_range)
        c_z = z_min + (nz3 // 2) * dz3
        nu_rz = (rel[:, 2] - c_z) / dz3
        torus = np.column_stack([2.0 * np.pi * nu_rx / px, 2.0 * np.pi * nu_ry / py,
                                 2.0 * np.pi * nu_rz / pz])
        self.plan = nu.NufftPlan((pz, py, px), eps, self.device)
        self.pts = self.plan.points(torus)
        # the frequencies of a group share one spreading pass (a tile's points and window
        # weights are staged once for up to 16 value sets); their fine grids stay within
        # _GROUP_FINE_BYTES
        per = 8 * self.n_illum * self.plan.fine_elems
        self.group_f = max(1, min(self.freqs.size, _GROUP_FINE_BYTES // per))
        self._fine = torch.empty((self.group_f * self.n_illum, self.plan.fine_elems),
                                 dtype=torch.complex64, device=self.device)

    def _lattice_spectrum(self, coeff_f, uhat3, n3, stream):
        nu.type1(self.plan, self.pts, coeff_f, self.n_illum, coeff_f.shape[-1], uhat3, n3,
                 self._fine, False, stream)

    def _lattice_spectra(self, coeff, f0, f1, uhat3g, n3, stream):
        nv = (f1 - f0) * self.n_illum
        vals = coeff[f0:f1].reshape(nv, coeff.shape[-1])
        nu.type1(self.plan, self.pts, vals, nv, coeff.shape[-1], uhat3g, n3, self._fine, False,
                 stream)


class Rsd3dEngine(_Lattice3dEngine):
    """Stage 1 by gridding the relay onto the virtual lattice (reconstruct.py:662-719):
    nearest or trilinear weights, duplicate targets summed, then cfft_n."""

    GRID_MSG = "rsd3d reconstructs onto a cuboid grid"

    def __init__(self, slices, grid, scatter="trilinear", z_pitch=None,
                 include_illumination=True, times=None, device=None, plane_range=None):
        _require(scatter in ("nearest", "trilinear"), "scatter must be 'nearest' or 'trilinear'")
        (rel, dz3, z_min, nz3, pz, z0, nu_rx, nu_ry, px, py, slab) = self._setup_lattice(
            slices, grid, z_pitch, include_illumination, times, device, plane_range)
        fx = nu_rx + px // 2
        fy = nu_ry + py // 2
        fz = (rel[:, 2] - z_min) / dz3 + (pz // 2 - nz3 // 2)
        n = fx.size
        if scatter == "nearest":
            ix = np.round(fx).astype(np.int64)[:, None]
            iy = np.round(fy).astype(np.int64)[:, None]
            iz = np.round(fz).astype(np.int64)[:, None]
            w = np.ones((n, 1))
        else:
            def corners(f):
                lo = np.floor(f).astype(np.int64)
                fr = f - lo
                return np.stack([lo, lo + 1], axis=1), np.stack([1.0 - fr, fr], axis=1)
            gx, wx = corners(fx)
            gy, wy = corners(fy)
            gz, wz = corners(fz)
            iz = np.broadcast_to(gz[:, :, None, None], (n, 2, 2, 2)).reshape(n, 8)
            iy = np.broadcast_to(gy[:, None, :, None], (n, 2, 2, 2)).reshape(n, 8)
            ix = np.broadcast_to(gx[:, None, None, :], (n, 2, 2, 2)).reshape(n, 8)
            w = (wz[:, :, None, None] * wy[:, None, :, None] * wx[:, None, None, :]).reshape(n, 8)
        for name, idx, bound in (("x", ix, px), ("y", iy, py), ("z", iz, pz)):
            assert idx.min() >= 0 and idx.max() < bound, \
                f"relay scatter indices escaped the {name} lattice"
        # lattice slot j holds centred lag j - n//2: its natural-order cell
        cell = ((((iz - pz // 2) % pz) * py + (iy - py // 2) % py) * px
                + (ix - px // 2) % px).ravel()
        pt = np.repeat(np.arange(n, dtype=np.int64), w.shape[1])
        order = np.argsort(cell, kind="stable")
        cell, pt, wf = cell[order], pt[order], w.ravel()[order]
        uniq, start = np.unique(cell, return_index=True)
        starts = np.append(start, cell.size).astype(np.int32)
        d = self.device
        self._csr = (torch.from_numpy(starts).to(d), torch.from_numpy(uniq.astype(np.int64)).to(d),
                     torch.from_numpy(pt.astype(np.int32)).to(d),
                     torch.from_numpy(wf.astype(np.float32)).to(d), int(uniq.size))
        self.n_relay = n

    def _lattice_spectrum(self, coeff_f, uhat3, n3, stream):
        st, cells, pts, wts, nc = self._csr
        uhat3.zero_()
        _lib.call("pf_scatter_csr", dev.ptr(st), dev.ptr(cells), dev.ptr(pts), dev.ptr(wts), nc,
                  dev.ptr(coeff_f), coeff_f.shape[-1], self.n_illum, dev.ptr(uhat3), n3,
                  dev.stream_ptr(stream))
        dev.fftn_natural(uhat3, (self.pz, self.py, self.px), self.n_illum, -1, 1.0, stream)


class Lattice3dSrsdEngine(GraphedRun):
    """The paper's "3D RSD / 3D NURSD + SRSD" ("the second stage is
    simply the standard RSD algorithm, so it can be replaced by SRSD"): stage 1 of nursd3d
    (reconstruct.py:741-760, 3D type-1 NUFFT) or rsd3d (:705-716, gridding) propagates the
    scattered 3D relay to the virtual plane z0 beyond its far face, on the lattice of the
    frustum's base (the lattice the cuboid grid supplies in nursd3d); the wave there,
    sampled on the base window (the centred crop of reconstruct.py:650-651), is a uniform
    relay at z0 whose coefficients srsd (:276-327) propagates onto the frustum, so the
    voxel pitch grows with depth.  No reference entry point exists; the oracle composes the
    same reference pieces (``oracle.lattice_srsd``)."""

    def __init__(self, slices, grid, stage1: str = "nursd3d", eps: float = 1e-6,
                 scatter: str = "trilinear", z_pitch: float | None = None, times=None,
                 include_illumination: bool = True, device=None):
        from .core import CuboidGrid, UniformGrid2D, UniformGrid3D, UniformRelay
        _require(_kind(grid) == "frustum", "this algorithm reconstructs onto a frustum grid")
        _require(stage1 in ("nursd3d", "rsd3d"), "stage 1 must be 'nursd3d' or 'rsd3d'")
        _nonplanar_relay(slices)
        self.device = device or dev.require_cuda()
        b = grid.base
        zs = np.asarray(grid.zs, dtype=np.float64)
        # stage-1 lattice: the frustum base's lateral lattice; its one plane at the nearest
        # frustum depth makes _lattice_3d check every depth against the far face z0
        lattice = CuboidGrid(UniformGrid3D(b.nx, b.ny, 1, b.dx, b.dy, 1.0, b.x0, b.y0,
                                           float(zs.min())))
        if stage1 == "nursd3d":
            self.stage1 = Nursd3dEngine(slices, lattice, eps, z_pitch, include_illumination,
                                        None, device=self.device)
        else:
            self.stage1 = Rsd3dEngine(slices, lattice, scatter, z_pitch, include_illumination,
                                      None, device=self.device)
        z0 = self.stage1.z0
        vrel = UniformRelay(UniformGrid2D(b.nx, b.ny, b.dx, b.dy, b.x0, b.y0, z0))
        meta = type("VirtualSlices", (), dict(frequencies=np.asarray(slices.frequencies),
                                              relay=vrel, illuminations=slices.illuminations))()
        self.stage2 = SrsdEngine(meta, grid, include_illumination, times, device=self.device)
        self.times, self.n_frames = self.stage2.times, self.stage2.n_frames
        self.n_voxels = self.stage2.n_voxels
        self.px, self.py = self.stage2.px, self.stage2.py
        F, I = self.stage2.freqs.size, self.stage2.n_illum
        self.window = torch.empty((F * I * b.ny * b.nx,), dtype=torch.complex64,
                                  device=self.device)

    def run(self, coeff, vol=None, stream=None):
        st1 = self.stage1
        F, I = st1.freqs.size, st1.n_illum
        b = self.stage2.g
        planes = st1.virtual_planes(coeff, stream)          # natural order [F*I][py][px]
        _lib.call("pf_crop_centered", dev.ptr(planes), F * I, st1.py, st1.px,
                  dev.ptr(self.window), b.ny, b.nx, dev.stream_ptr(stream))
        return self.stage2.run(self.window.view(F, I, b.ny * b.nx), vol, stream)


def nursd3d_srsd(slices, grid, eps: float = 1e-6, z_pitch: float | None = None, times=None,
                 threads: int = 1, include_illumination: bool = True):
    """3D NURSD stage 1 + SRSD stage 2 onto a frustum (see :class:`Lattice3dSrsdEngine`)."""
    eng = Lattice3dSrsdEngine(slices, grid, "nursd3d", eps, "trilinear", z_pitch, times,
                              include_illumination)
    return _volume(grid, eng.run(device_coefficients(slices)), eng.times)


def rsd3d_srsd(slices, grid, scatter: str = "trilinear", z_pitch: float | None = None,
               times=None, threads: int = 1, include_illumination: bool = True):
    """3D RSD (gridded) stage 1 + SRSD stage 2 onto a frustum (:class:`Lattice3dSrsdEngine`)."""
    eng = Lattice3dSrsdEngine(slices, grid, "rsd3d", 1e-6, scatter, z_pitch, times,
                              include_illumination)
    return _volume(grid, eng.run(device_coefficients(slices)), eng.times)


def nursd3d(slices, grid, eps: float = 1e-6, z_pitch: float | None = None, times=None,
            threads: int = 1, include_illumination: bool = True):
    """Scattered 3D relay -> cuboid (reconstruct.py:722-765)."""
    _require(_kind(grid) == "cuboid", "nursd3d reconstructs onto a cuboid grid")
    relay = _nonplanar_relay(slices)
    rel = np.asarray(relay.points.points)
    if float(rel[:, 2].max() - rel[:, 2].min()) == 0.0:
        flat = _FlatSlices(slices, rel)
        eng = Nursd1Engine(flat, grid, eps, include_illumination, times)
        return _volume(grid, eng.run(device_coefficients(slices)), eng.times)
    eng = Nursd3dEngine(slices, grid, eps, z_pitch, include_illumination, times)
    return _volume(grid, eng.run(device_coefficients(slices)), eng.times)


def rsd3d(slices, grid, scatter: str = "trilinear", z_pitch: float | None = None, times=None,
          threads: int = 1, include_illumination: bool = True):
    """3D relay -> cuboid by gridding + one 3D convolution (reconstruct.py:662-719)."""
    eng = Rsd3dEngine(slices, grid, scatter, z_pitch, include_illumination, times)
    return _volume(grid, eng.run(device_coefficients(slices)), eng.times)


# ---------------------------------------------------------------------------
# config 2: non-planar relay -> arbitrary voxels (3D NURSD stage 1 + NURSD-2)
# ---------------------------------------------------------------------------


class Nursd3dExplicitEngine(GraphedRun):
    """Non-planar relay -> explicit voxels: the paper's 3D NURSD + NURSD-2 fusion.

    The reference has no single entry point for this; it is composed
    from reference pieces exactly as SURVEY 8(d) specifies the config-2 oracle:
    the ``nursd3d`` stage 1 (reconstruct.py:741-760) propagates the scattered 3D
    relay to the virtual plane z0 on the lattice of the ``lattice`` cuboid
    (``_lattice_3d``, :594-621); that plane, in the lattice's centred slot
    order, becomes a uniform relay at z0 whose coefficients ``nursd2``
    (:413-459) reads out at the explicit voxels (every voxel plane beyond z0).
    Geometry-only planning (NUFFT plans, point buckets, pads) happens once here;
    ``run(coeff)`` is the per-capture work (and can be replayed as a CUDA graph).
    """

    def __init__(self, slices, grid, lattice, eps: float = 1e-6, z_pitch: float | None = None,
                 times=None, include_illumination: bool = True, device=None):
        from .core import UniformGrid2D, UniformRelay
        _require(_kind(grid) in ("explicit", "voxels"),
                 "nursd3d-explicit reconstructs onto explicit voxels")
        _require(_kind(lattice) == "cuboid", "the stage-1 lattice must be a cuboid grid")
        self.device = device or dev.require_cuda()
        self.stage1 = Nursd3dEngine(slices, lattice, eps, z_pitch, include_illumination, None,
                                    device=self.device)
        px, py = self.stage1.px, self.stage1.py
        vg = lattice.grid
        cx = vg.x0 + (vg.nx // 2) * vg.dx
        cy = vg.y0 + (vg.ny // 2) * vg.dy
        vrel = UniformRelay(UniformGrid2D(px, py, vg.dx, vg.dy, cx - (px // 2) * vg.dx,
                                          cy - (py // 2) * vg.dy, self.stage1.z0))
        meta = type("VirtualSlices", (), dict(frequencies=np.asarray(slices.frequencies),
                                              relay=vrel, illuminations=slices.illuminations))()
        # explicit planes: the plane readout; a voxel cloud (arbitrary depths, BASELINE
        # config 2's random voxel positions): the z-Chebyshev readout
        stage2 = Nursd2VoxelsEngine if _kind(grid) == "voxels" else Nursd2Engine
        self.stage2 = stage2(meta, grid, eps, times, include_illumination, self.device)
        self.times, self.n_frames = self.stage2.times, self.stage2.n_frames
        self.n_voxels = self.stage2.n_voxels
        self.px, self.py = px, py
        F, I = self.stage2.freqs.size, self.stage2.n_illum
        self.slot = torch.empty((F * I * py * px,), dtype=torch.complex64, device=self.device)

    def run(self, coeff, vol=None, stream=None):
        st1 = self.stage1
        F, I, px, py = st1.freqs.size, st1.n_illum, st1.px, st1.py
        planes = st1.virtual_planes(coeff, stream)
        # natural -> centred slot order (fftshift) and relay coefficient layout [F][I][py*px]
        _lib.call("pf_roll", dev.ptr(planes), dev.ptr(self.slot), F * I, 1, py, px, 0,
                  py - py // 2, px - px // 2, dev.stream_ptr(stream))
        return self.stage2.run(self.slot.view(F, I, py * px), vol, stream)


def nursd3d_explicit(slices, grid, lattice, eps: float = 1e-6, z_pitch: float | None = None,
                     times=None, threads: int = 1, include_illumination: bool = True):
    """Config-2 path (see :class:`Nursd3dExplicitEngine`)."""
    eng = Nursd3dExplicitEngine(slices, grid, lattice, eps, z_pitch, times, include_illumination)
    return _volume(grid, eng.run(device_coefficients(slices)), eng.times)
