"""CPU-only checks: size rules, plans, the C-ABI library surface, validation messages."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_2501_05244_b200 as pf
from paper_2501_05244_b200 import _fastlen, _lib
from paper_2501_05244_b200._device import radices_for

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_next_fast_len_kats():
    # pinned sizes of the reference pad rule (scipy's 11-smooth next_fast_len)
    for n, want in [(136, 140), (138, 140), (520, 525), (1023, 1024), (1034, 1050), (13, 14),
                    (169, 175), (1025, 1029), (2049, 2058), (1, 1), (2, 2), (128, 128)]:
        assert _fastlen.next_fast_len(n) == want


def test_next_fast_len_matches_scipy():
    sp = pytest.importorskip("scipy.fft")
    for n in range(1, 3000):
        assert _fastlen.next_fast_len(n) == sp.next_fast_len(n)


@pytest.mark.parametrize("n", [2, 3, 5, 7, 11, 16, 128, 140, 280, 512, 525, 1024, 1050, 2048, 2100])
def test_radices_multiply_back(n):
    r = radices_for(n)
    assert int(np.prod(r)) == n
    assert all(x in (2, 3, 4, 5, 7, 8, 11, 16) for x in r)


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    header = open(os.path.join(ROOT, "include", "pfgpu.h")).read()
    declared = set(re.findall(r"^(?:int|int64_t)\s+(pf_\w+)\(", header, flags=re.M))
    assert declared, "no declarations parsed"
    for name in declared:
        assert hasattr(lib, name), name
    assert declared <= set(_lib.exported_symbols())
    assert lib.pf_version() >= 1


def test_error_channel_without_device():
    lib = _lib.load()
    # argument errors are reported before any CUDA call
    rc = lib.pf_embed_centered(None, 1, 4, 4, 16, None, 2, 2, 0, None)
    assert rc < 0
    assert "pf_embed_centered" in _lib.last_error()


def _slices16():
    relay = pf.UniformRelay(pf.UniformGrid2D(16, 16, 0.02, 0.02, -0.15, -0.15, 0.0))
    ill = pf.PointList(np.array([[0.0, 0.0]]))
    coeff = np.ones((1, 256, 3), dtype=np.complex128)
    return pf.FrequencySlices(np.array([1e10, 1.1e10, 1.2e10]), coeff, relay, ill)


@pytest.mark.parametrize("grid,kw,match", [
    (pf.CuboidGrid(pf.UniformGrid3D(4, 4, 1, 0.03, 0.02, 0.1, -0.03, -0.01, 0.9)), {}, "pitch"),
    (pf.CuboidGrid(pf.UniformGrid3D(4, 4, 1, 0.02, 0.02, 0.1, -0.025, -0.01, 0.9)), {}, "origin"),
    (pf.CuboidGrid(pf.UniformGrid3D(4, 4, 2, 0.02, 0.02, 0.1, -0.03, -0.01, -0.05)), {},
     "beyond the relay"),
    (pf.CuboidGrid(pf.UniformGrid3D(4, 3, 2, 0.02, 0.02, 0.1, -0.03, -0.01, 0.85)),
     {"padding": "none"}, "padding="),
    (pf.CuboidGrid(pf.UniformGrid3D(4, 3, 2, 0.02, 0.02, 0.1, -0.03, -0.01, 0.85)),
     {"padding": "wrap"}, "padding"),
    (pf.ExplicitVoxels((pf.VoxelPlane(0.9, pf.PointList(np.array([[0.0, 0.0]]))),)), {}, "cuboid"),
    (pf.CuboidGrid(pf.UniformGrid3D(4, 3, 2, 0.02, 0.02, 0.1, -0.03, -0.01, 0.85)),
     {"times": np.zeros((2, 2))}, "times"),
])
def test_rsd_validation_messages(grid, kw, match):
    # reference test_reconstruct.py:148-183 (raised before any device work)
    with pytest.raises(pf.ValidationError, match=match):
        pf.rsd(_slices16(), grid, **kw)


def test_dispatcher_names_and_errors():
    assert pf.ALGORITHM_NAMES == ("rsd", "srsd", "nursd1", "nursd2", "nursd3", "rsd3d",
                                  "nursd3d", "srsd-nursd2")
    grid = pf.CuboidGrid(pf.UniformGrid3D(4, 3, 2, 0.02, 0.02, 0.1, -0.03, -0.01, 0.85))
    with pytest.raises(pf.ValidationError, match="unknown algorithm"):
        pf.reconstruct(_slices16(), grid, "fbp")
    ev = pf.ExplicitVoxels((pf.VoxelPlane(0.9, pf.PointList(np.array([[0.0, 0.0]]))),))
    with pytest.raises(pf.ValidationError, match="alpha"):
        pf.reconstruct(_slices16(), ev, "srsd-nursd2")


def test_build_kernel_matches_reference_kat():
    k = pf.build_kernel(0.04, 4096, 16e-12)
    assert k.n_freq == 95  # reference test_phasor.py:29-30
    with pytest.raises(pf.ValidationError):
        pf.build_kernel(0.04, 4096, 16e-12, threshold=0.9999999)


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    grid = pf.CuboidGrid(pf.UniformGrid3D(4, 3, 2, 0.02, 0.02, 0.1, -0.03, -0.01, 0.85))
    with pytest.raises(RuntimeError, match="CUDA"):
        pf.rsd(_slices16(), grid)


def test_rescale_to_torus_round_trip_and_errors():
    """Reference core.py:550-589: box -> [-pi, pi)^d and back; validation messages."""
    import paper_2501_05244_b200 as pf
    p = pf.PointList(np.array([[0.0, 1.0], [0.5, 1.9], [0.999, 1.0]]))
    t, m = pf.rescale_to_torus(p, [0.0, 1.0], [1.0, 2.0])
    assert np.all(t.points >= -np.pi) and np.all(t.points < np.pi)
    assert np.allclose(m.inverse(t.points), p.points, atol=1e-15)
    with pytest.raises(pf.ValidationError, match="inside the half-open box"):
        pf.rescale_to_torus(p, [0.0, 1.0], [0.5, 2.0])
    with pytest.raises(pf.ValidationError, match="positive extent"):
        pf.rescale_to_torus(p, [0.0, 1.0], [0.0, 2.0])


@pytest.mark.parametrize("shape,modes,nb", [((12, 10), (5, 6), 2), ((8, 12, 10), (3, 5, 6), 2),
                                            ((6, 9, 8), (6, 4, 3), 1), ((12, 10, 6), (5, 4, 3), 2),
                                            ((40, 54, 54), (20, 27, 27), 2)])
def test_fftn_pruned_line_sets(monkeypatch, shape, modes, nb):
    """The NUFFT's pruned fftn (host line-set logic) against numpy: type 1 keeps every
    kept output, type 2 (zero off the kept slots) is exact everywhere.  pf_fft_lines is
    emulated on the CPU buffer from its (inner, istr, ostr, estr) line indexing."""
    import torch
    from paper_2501_05244_b200 import _device as dev
    rng = np.random.default_rng(5)
    x = (rng.normal(size=(nb,) + shape) + 1j * rng.normal(size=(nb,) + shape)).astype(np.complex64)
    kept = [dev.kept_ranges(m, n) for m, n in zip(modes, shape)]
    t = torch.from_numpy(x.copy())
    flat = t.view(-1).numpy()
    base = t.data_ptr()

    def fake(name, p, planref, nl, inner, istr, *rest):
        if name == "pf_fft_lines":
            mid, mstr, (ostr, estr, direction, scale, stream) = 1 << 62, rest[0], (0,) + rest[1:]
        else:
            assert name == "pf_fft_lines3"
            mid, mstr, ostr, estr, direction, scale, stream = rest
        n = planref._obj.n
        off = (p - base) // 8
        for ln in range(nl):
            q = ln // inner
            idx = (off + (q // mid) * ostr + (q % mid) * mstr + (ln % inner) * istr
                   + np.arange(n) * estr)
            v = flat[idx].astype(np.complex128)
            flat[idx] = np.fft.fft(v) if direction < 0 else np.fft.ifft(v) * n
        return 0

    monkeypatch.setattr(dev._lib, "call", fake)
    axes = tuple(range(1, len(shape) + 1))
    sel = np.ix_(*[np.concatenate([np.arange(s0, s0 + ln) for s0, ln in k]) for k in kept])
    st = type("S", (), {"cuda_stream": 0})()   # no device: the emulated call ignores it
    dev.fftn_pruned(t, shape, nb, -1, kept, True, st)
    ref = np.fft.fftn(x.astype(np.complex128), axes=axes)
    for b in range(nb):
        np.testing.assert_allclose(flat.reshape((nb,) + shape)[b][sel], ref[b][sel], rtol=1e-4,
                                   atol=1e-4)
    # type 2: input zero off the kept slots, full inverse everywhere
    z = np.zeros_like(x)
    for b in range(nb):
        z[b][sel] = x[b][sel]
    t2 = torch.from_numpy(z.copy())
    flat = t2.view(-1).numpy()
    base = t2.data_ptr()
    dev.fftn_pruned(t2, shape, nb, +1, kept, False, st)
    ref2 = np.fft.ifftn(z.astype(np.complex128), axes=axes) * np.prod(shape)
    np.testing.assert_allclose(flat.reshape((nb,) + shape), ref2, rtol=1e-4, atol=1e-4)


@pytest.mark.parametrize("shape,modes,nz,nb", [
    ((12, 10), (5, 6), [[(3, 5)], [(0, 2), (7, 3)]], 2),                      # 2D, x arc wraps
    ((8, 12, 10), (3, 5, 6), [[(6, 2), (0, 1)], [(2, 7)], [(1, 6)]], 2),      # 3D, z arc wraps
    ((40, 54, 54), (20, 27, 27), [[(3, 30)], [(10, 26)], [(40, 14), (0, 12)]], 2)])
def test_fftn_pruned_skips_zero_lines(monkeypatch, shape, modes, nz, nb):
    """Type-1 line sets with the spreading's touched arcs (``nonzero``): the input is zero
    off the arcs, and every kept output still equals numpy's fftn."""
    import torch
    from paper_2501_05244_b200 import _device as dev
    rng = np.random.default_rng(6)
    x = np.zeros((nb,) + shape, dtype=np.complex64)
    idx = np.ix_(*[np.concatenate([np.arange(s0, s0 + ln) for s0, ln in r]) for r in nz])
    for b in range(nb):
        blk = x[b][idx].shape
        x[b][idx] = (rng.normal(size=blk) + 1j * rng.normal(size=blk)).astype(np.complex64)
    kept = [dev.kept_ranges(m, n) for m, n in zip(modes, shape)]
    t = torch.from_numpy(x.copy())
    flat = t.view(-1).numpy()
    base = t.data_ptr()
    lines = [0]

    def fake(name, p, planref, nl, inner, istr, *rest):
        if name == "pf_fft_lines":
            mid, mstr, ostr, estr = 1 << 62, rest[0], 0, rest[1]
        else:
            mid, mstr, ostr, estr = rest[:4]
        n = planref._obj.n
        off = (p - base) // 8
        lines[0] += nl
        for ln in range(nl):
            q = ln // inner
            i = (off + (q // mid) * ostr + (q % mid) * mstr + (ln % inner) * istr
                 + np.arange(n) * estr)
            flat[i] = np.fft.fft(flat[i].astype(np.complex128))
        return 0

    monkeypatch.setattr(dev._lib, "call", fake)
    st = type("S", (), {"cuda_stream": 0})()
    dev.fftn_pruned(t, shape, nb, -1, kept, True, st, nz)
    with_skip = lines[0]
    sel = np.ix_(*[np.concatenate([np.arange(s0, s0 + ln) for s0, ln in k]) for k in kept])
    ref = np.fft.fftn(x.astype(np.complex128), axes=tuple(range(1, len(shape) + 1)))
    for b in range(nb):
        np.testing.assert_allclose(flat.reshape((nb,) + shape)[b][sel], ref[b][sel], rtol=1e-4,
                                   atol=1e-4)
    lines[0] = 0
    t = torch.from_numpy(x.copy())
    flat = t.view(-1).numpy()
    base = t.data_ptr()
    dev.fftn_pruned(t, shape, nb, -1, kept, True, st)
    assert with_skip < lines[0]


def test_zcheb_slabs_interpolate_kernel_phases():
    """The depth slabs / Chebyshev nodes of the arbitrary-depth readout reproduce an
    exp(i k r)/r kernel sample at random depths to < 1e-6 (CPU: host planning only)."""
    from paper_2501_05244_b200.algorithms import zcheb_slabs
    k = 2 * np.pi / 0.055
    z = np.random.default_rng(5).uniform(1.0, 2.0, 20000)
    edges, node_z, slab, lw = zcheb_slabs(z, k)
    assert np.allclose(lw.sum(axis=1), 1.0)
    assert (z >= edges[slab] - 1e-12).all() and (z <= edges[slab + 1] + 1e-12).all()
    for rho in (0.0, 0.4, 1.1):
        def f(zz):
            r = np.sqrt(zz ** 2 + rho ** 2)
            return np.exp(1j * k * r) / r
        approx = (lw * f(node_z)[slab]).sum(axis=1)
        assert np.abs(approx - f(z)).max() / np.abs(f(z)).max() < 1e-6


def test_es_window_plan_meets_eps_against_direct_sums():
    """Host side of the exponential-of-semicircle NUFFT window (nufft.es_half_width /
    es_transform: half-width, beta, continuous deconvolution) in a float64 numpy type-1
    transform against the direct sum: within the requested eps (CPU: planning only)."""
    from paper_2501_05244_b200 import nufft as nu
    rng = np.random.default_rng(11)
    m = 48
    mr = 2 * m
    h = 2 * np.pi / mr
    x = rng.uniform(-np.pi, np.pi, 400)
    x[:40] = -np.pi + h * rng.integers(0, mr, 40)            # some points on fine-grid nodes
    c = rng.normal(size=400) + 1j * rng.normal(size=400)
    k = np.arange(m) - m // 2
    exact = (c[None, :] * np.exp(-1j * np.outer(k, x))).sum(axis=1)
    for eps, tol in ((1e-2, 3e-5), (1e-4, 3e-5), (1e-6, 3e-7), (1e-9, 1e-9)):
        w = nu.es_half_width(eps)
        assert w == max(3, -(-(int(np.ceil(np.log10(1 / eps))) + 2) // 2))
        beta = 2.30 * 2 * w
        ker = nu.es_transform(w, k * h)
        assert (ker > 0).all()
        xi = x - 2 * np.pi * np.floor(x / (2 * np.pi))
        i0 = np.floor(xi / h + 0.5).astype(int)
        offs = np.arange(-w, w + 1)
        z = ((i0[:, None] + offs[None, :]) * h - xi[:, None]) / (w * h)
        q = 1 - z * z
        wt = np.where(q > 0, np.exp(beta * (np.sqrt(np.maximum(q, 0)) - 1)), 0.0)
        fine = np.zeros(mr, complex)
        np.add.at(fine, (i0[:, None] + offs[None, :]) % mr, c[:, None] * wt)
        got = np.fft.fft(fine)[k % mr] / ker
        err = np.linalg.norm(got - exact) / np.linalg.norm(exact)
        assert err < tol and err < eps, (eps, w, err)


def test_stencil_window_and_touched_runs_host():
    """nufft.stencil_window (type-2: the fine cells any stencil touches) and
    NufftPoints.touched_runs (type-1: the arcs a spread grid is nonzero on), host logic on a
    stand-in plan: every stencil cell inside, shortest arcs, seam handled."""
    import types
    from paper_2501_05244_b200 import nufft as nu
    plan = types.SimpleNamespace(mrs=(1, 700, 540), w=4, dim=2)
    rng = np.random.default_rng(12)
    i0 = np.zeros((2000, 3), dtype=np.int64)
    i0[:, 1] = rng.integers(286, 414, 2000)                  # rows: one arc inside
    i0[:, 2] = rng.integers(-64, 64, 2000) % 540             # columns: an arc across the seam
    ps = types.SimpleNamespace(_i0_host=i0, plan=plan, _runs=None)
    c0, nc, r0, nr = nu.stencil_window(plan, [ps])
    assert (r0, nr) == (int(i0[:, 1].min()) - 4, int(i0[:, 1].max() - i0[:, 1].min()) + 9)
    assert c0 + nc > 540 and nc <= 128 + 9                   # wraps, and stays the short arc
    for a, (s0, n) in ((2, (c0, nc)), (1, (r0, nr))):
        mr = plan.mrs[a]
        cells = (i0[:, a][:, None] + np.arange(-4, 5)[None, :]) % mr
        assert (((cells - s0) % mr) < n).all()
    runs = nu.NufftPoints.touched_runs(ps)
    assert runs[0] == [(r0, nr)]
    assert runs[1] == [(0, c0 + nc - 540), (c0, 540 - c0)]
    # everything touched -> the whole axis
    i0[:, 1] = rng.integers(0, 700, 2000)
    assert nu.stencil_window(plan, [ps])[2:] == (0, 700)
