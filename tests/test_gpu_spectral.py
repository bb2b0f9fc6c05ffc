"""GPU transform primitives vs reference goldens (reference test_spectral.py semantics)."""

import numpy as np
import pytest

from oracle import pf_oracle as O
from golden_io import load

pytestmark = pytest.mark.gpu
TOL = 2e-6


def test_centred_ffts_golden():
    from paper_2501_05244_b200 import spectral as S
    d = load("spectral")
    for i in range(int(d["n_c"])):
        assert O.rel_l2(S.cfft_2d(d[f"c{i}_u"]), d[f"c{i}_fwd"]) < TOL
        assert O.rel_l2(S.cifft_2d(d[f"c{i}_u"]), d[f"c{i}_inv"]) < TOL


def test_centred_roundtrip_and_delta(rng):
    from paper_2501_05244_b200 import spectral as S
    for n in (1, 2, 3, 8, 15):
        u = rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))
        assert O.rel_l2(S.cifft_2d(S.cfft_2d(u)), u) < TOL
    for n in (4, 5, 9, 16):
        u = np.zeros(n, complex)
        u[n // 2] = 1.0
        assert O.rel_l2(S.cfft_n(u, (-1,)), np.ones(n)) < TOL


def test_sfft_golden():
    from paper_2501_05244_b200 import spectral as S
    d = load("spectral")
    for i in range(int(d["n_s"])):
        m, a, o = d[f"s{i}_args"]
        got = S.sfft_1d(d[f"s{i}_u"], a, int(o))
        assert O.rel_l2(got, d[f"s{i}_out"]) < 1e-5, (m, a, o)
    assert O.rel_l2(S.sfft_2d_centered(d["s2d_u"], 0.45, 0.8), d["s2d_out"]) < 1e-5


@pytest.mark.parametrize("window", ["es", "gaussian"])
def test_nufft_golden(monkeypatch, window):
    """Both windows against the reference's nufft1 / nufft2 outputs: the reference's own
    Gaussian stencil and the exponential-of-semicircle window under the same eps."""
    from paper_2501_05244_b200 import nufft as nu
    from paper_2501_05244_b200 import spectral as S
    monkeypatch.setattr(nu, "DEFAULT_WINDOW", window)
    d = load("spectral")
    for i in range(int(d["n_n"])):
        modes = tuple(int(m) for m in d[f"n{i}_modes"])
        eps = float(d[f"n{i}_eps"])
        t1 = S.nufft1(d[f"n{i}_pts"], d[f"n{i}_vals"], modes, eps)
        assert O.rel_l2(t1, d[f"n{i}_t1"]) < max(1e-5, 10 * eps), modes
        t2 = S.nufft2(d[f"n{i}_coeff"], d[f"n{i}_pts"], eps)
        assert O.rel_l2(t2, d[f"n{i}_t2"]) < max(1e-5, 10 * eps), modes


@pytest.mark.parametrize("window", ["es", "gaussian"])
def test_nufft_on_grid_exact_and_adjoint(rng, monkeypatch, window):
    """Points on fine-grid nodes: exact with the reference's Gaussian stencil (its discrete
    deconvolution), within the eps contract with the default window (continuous
    deconvolution); type 1 and type 2 are adjoint with either."""
    from paper_2501_05244_b200 import nufft as nu
    from paper_2501_05244_b200 import spectral as S
    monkeypatch.setattr(nu, "DEFAULT_WINDOW", window)
    m = 8
    j = rng.integers(0, m, size=20)
    pts = (-np.pi + 2 * np.pi * j / m).reshape(-1, 1)
    vals = rng.normal(size=20) + 1j * rng.normal(size=20)
    err = O.rel_l2(S.nufft1(pts, vals, (m,), 1e-4), O.nudft1(pts, vals, (m,)))
    assert err < (TOL if window == "gaussian" else 0.2 * 1e-4), err
    modes = (9, 7)
    p = rng.uniform(-np.pi, np.pi, size=(31, 2))
    v = rng.normal(size=31) + 1j * rng.normal(size=31)
    c = rng.normal(size=modes) + 1j * rng.normal(size=modes)
    lhs = np.vdot(S.nufft1(p, v, modes, 1e-10), c)
    rhs = np.vdot(v, S.nufft2(c, p, 1e-10))
    assert abs(lhs - rhs) / abs(lhs) < 1e-5


def test_nufft2_3d_vs_direct_sum(rng):
    """3D type 2 (reference spectral.py:361-381 supports 1-3 D) against the direct sum."""
    from paper_2501_05244_b200 import spectral as S
    modes = (6, 10, 9)
    c = rng.normal(size=modes) + 1j * rng.normal(size=modes)
    p = rng.uniform(-np.pi, np.pi, size=(57, 3))
    assert O.rel_l2(S.nufft2(c, p, 1e-6), O.nudft2(c, p)) < 1e-5


def test_plain_2d_ffts(rng):
    """fft_2d / ifft_2d / dft_2d / idft_2d (reference spectral.py:77-104), batched last axes."""
    from paper_2501_05244_b200 import spectral as S
    u = rng.normal(size=(3, 12, 10)) + 1j * rng.normal(size=(3, 12, 10))
    assert O.rel_l2(S.fft_2d(u), np.fft.fft2(u)) < 1e-6
    assert O.rel_l2(S.ifft_2d(u), np.fft.ifft2(u)) < 1e-6
    assert O.rel_l2(S.dft_2d(u[0]), np.fft.fft2(u[0])) < 1e-6
    assert O.rel_l2(S.idft_2d(u[1]), np.fft.ifft2(u[1])) < 1e-6


@pytest.mark.parametrize("m,eps", [(128, 1e-6), (256, 1e-4), (1024, 1e-6)])
def test_type1_register_finish_vs_oracle(rng, m, eps):
    """Split register-FFT type-1 finish (pf_nufft_type1_finish_pow2, mr = 2m) against the
    float64 oracle nufft1 (reference spectral.py:336-358) and the generic fftn + deconv."""
    import torch
    from paper_2501_05244_b200 import nufft as nu
    dev = torch.device("cuda")
    L, nv = 2000, 3
    pts = rng.uniform(-np.pi, np.pi, size=(L, 2))
    pts[:500] = -np.pi + 2 * np.pi * rng.integers(0, m, size=(500, 2)) / m   # on-lattice nodes
    vals = (rng.normal(size=(nv, L)) + 1j * rng.normal(size=(nv, L))).astype(np.complex64)
    plan = nu.NufftPlan((m, m), eps, dev)
    assert plan.pow2_finish and plan.mrs[1:] == (2 * m, 2 * m)
    p = plan.points(pts)
    v = torch.from_numpy(vals).to(dev)
    out = torch.full((nv, m, m), complex(np.nan, np.nan), dtype=torch.complex64, device=dev)
    nu.type1(plan, p, v, nv, L, out, m * m, transpose=True)
    plan.pow2_finish = False
    gen = torch.empty_like(out)
    nu.type1(plan, p, v, nv, L, gen, m * m, transpose=True)
    got, ref_gpu = out.cpu().numpy(), gen.cpu().numpy()
    assert O.rel_l2(got, ref_gpu) < 2e-6
    for i in range(nv if m <= 256 else 1):
        ref = O.nufft1(pts, vals[i].astype(np.complex128), (m, m), eps)
        # natural-order modes, transposed [x][y]; the oracle returns centred [y][x]
        ref_nat = np.fft.ifftshift(ref).T
        # the oracle is the reference's Gaussian stencil, the plan the default window: both
        # approximate the same sums within eps (measured 3e-7 at eps = 1e-6, 7e-6 at 1e-4)
        assert O.rel_l2(got[i], ref_nat) < max(2e-6, 0.2 * eps)


@pytest.mark.parametrize("window,eps,tol", [("es", 1e-6, 1e-6), ("es", 1e-4, 3e-5), ("es", 1e-2, 3e-5),
                                            ("es", 1e-9, 1e-6), ("gaussian", 1e-6, 1e-6)])
def test_nufft_windows_vs_direct_sums(rng, window, eps, tol):
    """Type 1 and type 2 in 2D against the direct sums (no NUFFT in the reference value):
    the window's own error, which the eps contract bounds; float32 arithmetic floors it
    near 3e-7."""
    import torch
    from paper_2501_05244_b200 import nufft as nu
    from paper_2501_05244_b200 import spectral as S
    dev = torch.device("cuda")
    modes = (40, 36)
    pts = rng.uniform(-np.pi, np.pi, size=(300, 2))
    pts[:40] = -np.pi + 2 * np.pi * rng.integers(0, 72, size=(40, 2)) / 72   # fine-grid nodes
    vals = rng.normal(size=300) + 1j * rng.normal(size=300)
    coeff = rng.normal(size=modes) + 1j * rng.normal(size=modes)
    plan = nu.NufftPlan(modes, eps, dev, window=window)
    assert plan.w == (nu.es_half_width(eps) if window == "es" else
                      max(2, int(np.ceil(np.log10(1 / eps))) + 2))
    import unittest.mock as um
    with um.patch.object(nu, "DEFAULT_WINDOW", window):
        t1 = S.nufft1(pts, vals, modes, eps)
        t2 = S.nufft2(coeff, pts, eps)
    assert O.rel_l2(t1, O.nudft1(pts, vals, modes)) < tol
    assert O.rel_l2(t2, O.nudft2(coeff, pts)) < tol


@pytest.mark.parametrize("modes,nv,split", [
    ((350, 350), 3, True),     # fine 700 = 2 x 350: two 350-point register FFTs per line
    ((64, 64), 2, False),      # fine 128: Stockham
    ((45, 63), 2, False),      # odd modes, fine 90 x 126
    ((140, 140), 5, True),     # fine 280 = 2 x 140
    ((175, 175), 2, True),     # odd modes with a split: fine 350 = 2 x 175
    ((70, 350), 2, True)])     # split along x only (70 = 35 x 2 has no register FFT)
def test_type2_start_fused_equals_place_and_pruned_fft(rng, monkeypatch, modes, nv, split):
    """pf_nufft_type2_start_2d (place + inverse fine-grid FFT in two fused passes) writes
    the same fine grid as pf_nufft_place + the pruned line passes: bit for bit with the
    full-length passes, to float32 rounding when a fine line (mr = 2 m = 70 L) runs as two
    half-length transforms of its modes."""
    import torch
    from paper_2501_05244_b200 import nufft as nu
    plan = nu.NufftPlan(modes, 1e-6, torch.device("cuda"))
    my, mx = modes
    S = torch.from_numpy((rng.normal(size=(nv, my * mx)) + 1j * rng.normal(size=(nv, my * mx)))
                         .astype(np.complex64)).cuda()
    fine_a = torch.full((nv, plan.fine_elems), complex(np.nan, np.nan), dtype=torch.complex64,
                        device="cuda")
    fine_b = torch.empty_like(fine_a)
    monkeypatch.setattr(nu, "_T2_FUSED", True)
    nu.place_and_inverse(plan, S, nv, my * mx, fine_a)
    monkeypatch.setattr(nu, "_T2_FUSED", False)
    nu.place_and_inverse(plan, S, nv, my * mx, fine_b)
    torch.cuda.synchronize()
    if split:
        assert bool(torch.isfinite(torch.view_as_real(fine_a)).all())
        d = (fine_a - fine_b).abs().pow(2).sum().sqrt() / fine_b.abs().pow(2).sum().sqrt()
        assert float(d) < 1e-6, float(d)
    else:
        assert torch.equal(fine_a, fine_b)
    # and it is the inverse DFT of the placed spectrum
    mry, mrx = plan.mrs[1], plan.mrs[2]
    ky, kx = (k.cpu().numpy().astype(np.float64) for k in plan.kers[1:])
    grid = np.zeros((mry, mrx), complex)
    s0 = S[0].cpu().numpy().reshape(my, mx).astype(complex)
    cy = np.arange(my) - my // 2
    cx = np.arange(mx) - mx // 2
    sc = s0[np.ix_(cy % my, cx % mx)] / np.outer(ky, kx)
    grid[np.ix_(cy % mry, cx % mrx)] = sc
    ref = np.fft.ifft2(grid) * mry * mrx
    got = fine_a[0].cpu().numpy().reshape(mry, mrx)
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-5


@pytest.mark.parametrize("modes,win", [((350, 350), (632, 136, 282, 140)),   # columns wrap the seam
                                       ((140, 140), (10, 50, 250, 60)),      # rows wrap the seam
                                       ((70, 350), (100, 200, 0, 140))])     # x split only
def test_type2_start_window(rng, modes, win):
    """pf_nufft_type2_start_2d_win: the fine cells inside the window are bit-identical to the
    full start and (where the column pass is split) cells in columns outside it stay
    unwritten -- the readout stencils never touch them (nufft.stencil_window)."""
    import torch
    from paper_2501_05244_b200 import nufft as nu
    plan = nu.NufftPlan(modes, 1e-6, torch.device("cuda"))
    my, mx = modes
    mry, mrx = plan.mrs[1], plan.mrs[2]
    nv = 3
    S = torch.from_numpy((rng.normal(size=(nv, my * mx)) + 1j * rng.normal(size=(nv, my * mx)))
                         .astype(np.complex64)).cuda()
    full = torch.empty((nv, plan.fine_elems), dtype=torch.complex64, device="cuda")
    part = torch.full_like(full, complex(np.nan, np.nan))
    nu.place_and_inverse(plan, S, nv, my * mx, full)
    nu.place_and_inverse(plan, S, nv, my * mx, part, window=win)
    torch.cuda.synchronize()
    c0, nc, r0, nr = win
    cols = (c0 + np.arange(nc)) % mrx
    rows = (r0 + np.arange(nr)) % mry
    f = full.cpu().numpy().reshape(nv, mry, mrx)
    g = part.cpu().numpy().reshape(nv, mry, mrx)
    inside = np.ix_(np.arange(nv), rows, cols)
    assert np.array_equal(f[inside], g[inside])
    if mry == 2 * my and my % 35 == 0 and my // 35 in (4, 5, 8, 10, 15, 20, 30):   # split column pass
        out_cols = np.setdiff1d(np.arange(mrx), cols)
        out_rows = np.setdiff1d(np.arange(mry), np.concatenate([np.arange(my - my // 2),
                                                                np.arange(mry - my // 2, mry)]))
        assert np.isnan(g[np.ix_(np.arange(nv), out_rows, out_cols)]).all()


def test_stencil_window_covers_every_tap(rng):
    """nufft.stencil_window holds every stencil cell of every point, across the seam too."""
    import torch
    from paper_2501_05244_b200 import nufft as nu
    plan = nu.NufftPlan((350, 350), 1e-6, torch.device("cuda"))
    pts = np.column_stack([rng.uniform(-0.4, 0.7, 500), rng.uniform(2.6, 3.6, 500)])
    pts[:, 1] = (pts[:, 1] + np.pi) % (2 * np.pi) - np.pi          # y straddles +-pi
    P = plan.points(pts)
    c0, nc, r0, nr = nu.stencil_window(plan, [P])
    assert nc < 300 and nr < 200
    for a, (s0, n) in ((2, (c0, nc)), (1, (r0, nr))):
        mr = plan.mrs[a]
        cells = (P._i0_host[:, a][:, None] + np.arange(-plan.w, plan.w + 1)[None, :]) % mr
        assert (((cells - s0) % mr) < n).all()
