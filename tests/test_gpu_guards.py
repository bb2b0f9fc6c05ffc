"""Memory-safety checks in place of compute-sanitizer (closed on this GPU pool: see
profiles/r2_compute_sanitizer_closed.txt).

* Read-before-write: every engine workspace is filled with NaN after a first run; a second
  run must give the bitwise-identical volume (any read of a stale or unwritten workspace
  element would carry NaN or a different value into it).
* Out-of-bounds writes: the volume is a view into a larger buffer whose guard bands hold a
  sentinel pattern; the guard bands must be untouched after the run.
Covered: rsd (frequency-batched and per-frequency A / fused B / C-Horner launches, 1 and 2
illuminations, video frames), srsd (Bluestein register passes), nursd1 (type-1 spreading
and register finish), nursd2 (type-2 readout), and K1.
"""

import importlib

import numpy as np
import pytest
import torch

import paper_2501_05244_b200 as pf
from paper_2501_05244_b200.algorithms import Nursd1Engine, Nursd2Engine, SrsdEngine
from paper_2501_05244_b200.phasor import device_coefficients

pytestmark = pytest.mark.gpu
R = importlib.import_module("paper_2501_05244_b200.reconstruct")

_WS = ("ws_a_l", "ws_b_l", "ws_o_l", "uhat", "uhat_l", "xbuf_l", "fine", "spec", "_fb_ws_a",
       "_fb_ws_b", "_fine", "slot")
_SUB = ("prop", "ro", "stage1", "stage2")
GUARD = 1 << 16


def _poison(obj, seen=None):
    seen = seen if seen is not None else set()
    if id(obj) in seen:
        return 0
    seen.add(id(obj))
    n = 0
    for name in _WS:
        v = getattr(obj, name, None)
        for t in (v if isinstance(v, list) else list(v.values()) if isinstance(v, dict) else [v]):
            if isinstance(t, torch.Tensor) and t.is_cuda and t.is_floating_point() | t.is_complex():
                (torch.view_as_real(t) if t.is_complex() else t).fill_(float("nan"))
                n += 1
    for name in _SUB:
        sub = getattr(obj, name, None)
        if sub is not None:
            n += _poison(sub, seen)
    return n


def _guarded(n_frames, n_vox):
    buf = torch.empty((n_frames * n_vox + 2 * GUARD,), dtype=torch.complex64, device="cuda")
    sentinel = torch.complex(torch.full((GUARD,), 1234.5, device="cuda"),
                             torch.full((GUARD,), -6789.25, device="cuda"))
    buf[:GUARD] = sentinel
    buf[-GUARD:] = sentinel
    return buf, buf[GUARD:GUARD + n_frames * n_vox].view(n_frames, n_vox), sentinel


def _check(eng, coeff, n_frames, n_vox):
    first = eng.run(coeff).clone()
    assert torch.isfinite(torch.view_as_real(first)).all()
    assert _poison(eng) >= 1
    buf, vol, sentinel = _guarded(n_frames, n_vox)
    out = eng.run(coeff, vol)
    torch.cuda.synchronize()
    assert out.data_ptr() == vol.data_ptr()
    assert torch.equal(buf[:GUARD], sentinel) and torch.equal(buf[-GUARD:], sentinel)
    assert torch.equal(vol, first), "result changed after poisoning the workspaces"


def _slices(rng, relay, F=5, n_ill=1):
    D = relay.count
    freqs = 2 * np.pi * 299792458.0 / 0.06 * (1 + 0.03 * np.arange(F))
    c = rng.normal(size=(n_ill, D, F)) + 1j * rng.normal(size=(n_ill, D, F))
    ill = pf.PointList(rng.uniform(-0.2, 0.2, size=(n_ill, 2)))
    return pf.FrequencySlices(freqs, c, relay, ill)


def _lattice(n):
    p = 2.0 / n
    return pf.UniformGrid2D(n, n, p, p, -1 + p / 2, -1 + p / 2, 0.0)


@pytest.mark.parametrize("n,nz,n_ill,video,fbatch,F", [
    (64, 6, 1, False, True, 5), (64, 6, 1, False, False, 5), (64, 5, 2, False, False, 5),
    (64, 5, 1, False, False, 70),
    (128, 4, 1, True, False, 5), (96, 3, 1, False, False, 5), (512, 3, 1, False, False, 5)])
def test_rsd_workspaces_and_guards(rng, monkeypatch, n, nz, n_ill, video, fbatch, F):
    if not fbatch:
        monkeypatch.setattr(R, "_FBATCH_BYTES", 0)
    g = _lattice(n)
    sl = _slices(rng, pf.UniformRelay(g), F=F, n_ill=n_ill)
    grid = pf.CuboidGrid(pf.UniformGrid3D(n, n, nz, g.dx, g.dy, 0.2, g.x0, g.y0, 0.5))
    times = np.array([0.0, 1e-10, 2e-10]) if video else None
    eng = R.RsdEngine(sl, grid, times=times)
    _check(eng, device_coefficients(sl), eng.n_frames, eng.n_voxels)


@pytest.mark.parametrize("n", [32, 64])
def test_srsd_workspaces_and_guards(rng, n):
    g = _lattice(n)
    sl = _slices(rng, pf.UniformRelay(g))
    zs = np.linspace(0.6, 1.8, 5)
    eng = SrsdEngine(sl, pf.FrustumGrid(g, zs, zs[0] / zs, zs[0] / zs))
    _check(eng, device_coefficients(sl), eng.n_frames, eng.n_voxels)


def test_nursd1_workspaces_and_guards(rng):
    pts = rng.uniform(-1, 1, size=(2000, 2))
    sl = _slices(rng, pf.NonUniformPlanarRelay(pf.PointList(pts), 0.0))
    g = _lattice(64)
    grid = pf.CuboidGrid(pf.UniformGrid3D(64, 64, 4, g.dx, g.dy, 0.2, g.x0, g.y0, 0.5))
    eng = Nursd1Engine(sl, grid)
    _check(eng, device_coefficients(sl), eng.n_frames, eng.n_voxels)


def test_nursd2_workspaces_and_guards(rng):
    g = _lattice(48)
    sl = _slices(rng, pf.UniformRelay(g), F=3)
    planes = tuple(pf.VoxelPlane(z, pf.PointList(rng.uniform(-0.6, 0.6, size=(300, 2))))
                   for z in (0.6, 0.8, 1.1))
    eng = Nursd2Engine(sl, pf.ExplicitVoxels(planes))
    _check(eng, device_coefficients(sl), eng.n_frames, eng.n_voxels)


def test_k1_output_guards(rng):
    T, D = 2048, 3000
    k = pf.build_kernel(0.06, T, 8e-12)
    hist = torch.rand((1, D, T), device="cuda")
    ref = pf.to_frequency_device(hist, k, 1e-10)
    F = k.n_freq
    buf = torch.full((F * D + 2 * GUARD,), complex(3.0, -7.0), dtype=torch.complex64,
                     device="cuda")
    from paper_2501_05244_b200.phasor import TemporalPlan
    out = buf[GUARD:GUARD + F * D].view(F, D)
    TemporalPlan(k, 1e-10, torch.device("cuda")).run(hist.view(D, T), out)
    torch.cuda.synchronize()
    assert torch.equal(out, ref.view(F, D))
    assert bool((buf[:GUARD] == complex(3.0, -7.0)).all())
    assert bool((buf[-GUARD:] == complex(3.0, -7.0)).all())
