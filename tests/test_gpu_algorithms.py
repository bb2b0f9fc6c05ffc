"""GPU parity of srsd / nursd1 / nursd2 / nursd3 / srsd_nursd2 / nursd3d / rsd3d vs reference
goldens + oracle."""

import numpy as np
import pytest
import torch

import paper_2501_05244_b200 as pf
from oracle import pf_oracle as O
from golden_io import case_call, grid_from, load, slices_from

pytestmark = pytest.mark.gpu
TOL = 1e-4

CASES = ["chain_srsd_unit", "chain_srsd_08", "chain_nursd1", "chain_nursd2", "chain_nursd3",
         "chain_hybrid", "chain_nursd3d_flat", "nursd1_random", "nursd2_random", "nursd3_random",
         "hybrid_random", "srsd_linear16", "srsd_aniso16", "nursd3d_curved", "rsd3d_curved_tri",
         "rsd3d_curved_near"]


@pytest.fixture(params=["es", "gaussian"])
def window(request, monkeypatch):
    """Run under both NUFFT windows: the default exponential of semicircle and the
    reference's Gaussian stencil (Python plans and the C entry points' planner)."""
    from paper_2501_05244_b200 import _lib
    from paper_2501_05244_b200 import nufft as nu
    monkeypatch.setattr(nu, "DEFAULT_WINDOW", request.param)
    prev = _lib.call("pf_nufft_window", 1 if request.param == "es" else 0)
    yield request.param
    _lib.call("pf_nufft_window", prev)


@pytest.mark.parametrize("name", CASES)
def test_algorithm_golden(name, window):
    d = load(f"rec_{name}")
    sl, grid = slices_from(d), grid_from(d)
    alg, kw = case_call(name)
    vol = pf.reconstruct(sl, grid, alg, **kw)
    assert O.rel_l2(vol.field, d["field"]) < TOL, name
    if grid.kind != "explicit":
        a = np.abs(vol.field.reshape(grid.shape)).max(axis=0)
        b = np.abs(d["field"].reshape(grid.shape)).max(axis=0)
        assert int(np.argmax(a)) == int(np.argmax(b))
    if "video" in d:
        v = pf.srsd(sl, grid, times=np.array([0.0, 5e-10]))
        assert O.rel_l2(v.field, d["video"]) < TOL


def test_degeneracy_chain_against_rsd():
    """Every variant on degenerate input equals rsd (reference test_reconstruct.py:191-239)."""
    ref = load("rec_chain_rsd")["field"]
    for name in ["chain_srsd_unit", "chain_nursd1", "chain_nursd2", "chain_nursd3", "chain_hybrid"]:
        d = load(f"rec_{name}")
        alg, kw = case_call(name)
        vol = pf.reconstruct(slices_from(d), grid_from(d), alg, **kw)
        assert O.rel_l2(vol.field, ref) < TOL, name


def _rand_slices(rng, relay, n_freq=3, n_ill=1, lam=0.06):
    w0 = 2 * np.pi * 299792458.0 / lam
    freqs = w0 * (1.0 + 0.03 * np.arange(n_freq))
    coeff = rng.normal(size=(n_ill, relay.count, n_freq)) + 1j * rng.normal(size=(n_ill, relay.count, n_freq))
    ill = pf.PointList(rng.uniform(-0.3, 0.3, size=(n_ill, 2)))
    return pf.FrequencySlices(freqs, coeff, relay, ill)


def test_nursd1_c1_like(rng, window):
    """Config-1 shape (i.i.d. relay points, P=140 from the reference pad rule), reduced size."""
    pts = rng.uniform(-1.0, 1.0, size=(4096, 2))
    sl = _rand_slices(rng, pf.NonUniformPlanarRelay(pf.PointList(pts), 0.0), n_freq=2)
    p = 2.0 / 64
    grid = pf.CuboidGrid(pf.UniformGrid3D(64, 64, 3, p, p, 0.5, -1 + p / 2, -1 + p / 2, 0.5))
    vol = pf.nursd1(sl, grid)
    ref = O.nursd1(sl, grid)
    assert O.rel_l2(vol.field, ref) < TOL


@pytest.mark.parametrize("n_ill", [1, 2])
def test_generic_fbatch_matches_per_frequency(rng, monkeypatch, n_ill):
    """Frequency-batched Stockham path (pf_prop_fbatch_generic, P = 140) reproduces the
    per-frequency launches bit for bit, and both match the oracle."""
    import importlib
    R = importlib.import_module("paper_2501_05244_b200.reconstruct")
    from paper_2501_05244_b200.algorithms import Nursd1Engine
    pts = rng.uniform(-1.0, 1.0, size=(2048, 2))
    sl = _rand_slices(rng, pf.NonUniformPlanarRelay(pf.PointList(pts), 0.0), n_freq=4,
                      n_ill=n_ill)
    p = 2.0 / 64
    grid = pf.CuboidGrid(pf.UniformGrid3D(64, 64, 5, p, p, 0.3, -1 + p / 2, -1 + p / 2, 0.5))
    eng = Nursd1Engine(sl, grid)
    assert not eng.prop.transposed and eng.px == 140
    eng.prop.onchip = False   # the Stockham path (the on-chip kernel: test_gpu_onchip.py)
    coeff = pf.phasor.device_coefficients(sl)
    assert eng.prop.fbatch_ok(sl.n_freq, 1)
    batched = eng.run(coeff).clone()
    monkeypatch.setattr(R, "_FBATCH_GENERIC", False)
    assert not eng.prop.fbatch_ok(sl.n_freq, 1)
    per_f = eng.run(coeff)
    torch.cuda.synchronize()
    assert torch.equal(batched, per_f)
    ref = O.nursd1(sl, grid)
    assert O.rel_l2(batched.cpu().numpy().reshape(ref.shape), ref) < TOL


def test_nursd1_on_lattice_register_path(rng):
    """Lattice-subsampled relay (config-4 NURSD variant, F4): P-independent, fast pads."""
    n = 64
    p = 2.0 / n
    g = pf.UniformGrid2D(n, n, p, p, -1 + p / 2, -1 + p / 2, 0.0)
    xy = pf.grid_coordinates(g).points
    keep = rng.random(xy.shape[0]) < 0.5
    sl = _rand_slices(rng, pf.NonUniformPlanarRelay(pf.PointList(xy[keep]), 0.0), n_freq=2)
    grid = pf.CuboidGrid(pf.UniformGrid3D(n, n, 3, p, p, 0.5, g.x0, g.y0, 0.5))
    from paper_2501_05244_b200.algorithms import Nursd1Engine
    eng = Nursd1Engine(sl, grid)
    assert eng.prop.transposed and eng.px == 128
    vol = pf.nursd1(sl, grid)
    # equals rsd on the zero-filled lattice (reference test_acceptance.py:174-176)
    full = np.zeros((1, n * n, 2), complex)
    full[:, keep, :] = sl.coefficients
    slu = pf.FrequencySlices(sl.frequencies, full, pf.UniformRelay(g), sl.illuminations)
    assert O.rel_l2(vol.field, O.rsd(slu, grid)) < TOL
    assert O.rel_l2(vol.field, O.nursd1(sl, grid)) < TOL


@pytest.mark.parametrize("n,frames", [(64, False), (128, True)])
def test_srsd_frustum_vs_oracle(rng, n, frames):
    """Config-3 shape (linear frustum, P = next_fast_len(2N) power of two), reduced size."""
    p = 2.0 / n
    g = pf.UniformGrid2D(n, n, p, p, -1 + p / 2, -1 + p / 2, 0.0)
    sl = _rand_slices(rng, pf.UniformRelay(g), n_freq=2, lam=0.08)
    zs = np.linspace(1.0, 3.0, 3)
    grid = pf.FrustumGrid(g, zs, zs[0] / zs, zs[0] / zs)
    times = np.array([0.0, 3e-10]) if frames else None
    vol = pf.srsd(sl, grid, times=times)
    ref = O.srsd(sl, grid, times=times)
    assert O.rel_l2(vol.field, ref) < TOL


def test_nursd2_offlattice_voxels(rng, window):
    n = 24
    p = 0.02
    g = pf.UniformGrid2D(n, n, p, p, -(n - 1) * p / 2, -(n - 1) * p / 2, 0.0)
    sl = _rand_slices(rng, pf.UniformRelay(g), n_freq=2, n_ill=2)
    planes = tuple(pf.VoxelPlane(z, pf.PointList(rng.uniform(-0.2, 0.2, size=(50, 2))))
                   for z in (0.7, 0.9))
    ev = pf.ExplicitVoxels(planes)
    vol = pf.nursd2(sl, ev)
    assert O.rel_l2(vol.field, O.nursd2(sl, ev)) < TOL


def test_nursd2_trimmed_readout_matches_full_stencil(rng, monkeypatch):
    """The Gaussian readout for w = 8 keeps 16 x 16 of the 17 x 17 taps (the far edge tap of
    an axis weighs <= 6.5e-9 of the centre tap): against the full stencil the volume moves
    by less than float32 rounding of the sum, and both match the oracle alike."""
    from paper_2501_05244_b200 import _lib
    from paper_2501_05244_b200 import nufft as nu
    monkeypatch.setattr(nu, "DEFAULT_WINDOW", "gaussian")
    n = 32
    p = 0.02
    g = pf.UniformGrid2D(n, n, p, p, -(n - 1) * p / 2, -(n - 1) * p / 2, 0.0)
    sl = _rand_slices(rng, pf.UniformRelay(g), n_freq=3, n_ill=1)
    pts = rng.uniform(-0.25, 0.25, size=(4000, 2))
    pts[:200] = np.round(pts[:200] / p) * p          # some voxels on relay-lattice nodes
    ev = pf.ExplicitVoxels((pf.VoxelPlane(0.6, pf.PointList(pts[:2000])),
                            pf.VoxelPlane(0.8, pf.PointList(pts[2000:]))))
    ref = O.nursd2(sl, ev)
    prev = _lib.call("pf_nufft_interp_mode", 2)
    try:
        trimmed = pf.nursd2(sl, ev).field
        _lib.call("pf_nufft_interp_mode", 1)
        full = pf.nursd2(sl, ev).field
    finally:
        _lib.call("pf_nufft_interp_mode", prev)
    assert O.rel_l2(trimmed, full) < 2e-7
    e_t, e_f = O.rel_l2(trimmed, ref), O.rel_l2(full, ref)
    assert e_t < 2e-6 and e_f < 2e-6 and abs(e_t - e_f) < 2e-7, (e_t, e_f)


@pytest.mark.parametrize("n_freq", [3, 16, 20])
def test_nursd2_fused_frequency_readout_matches_per_frequency(rng, monkeypatch, n_freq):
    """The readout over all frequencies in one launch (frequency-interleaved fine grids, 16
    per group: 3 = padded slots, 20 = two groups) against the per-frequency launches and the
    oracle; voxels up to the edge of the reference pad."""
    import importlib
    A = importlib.import_module("paper_2501_05244_b200.algorithms")
    n = 32
    p = 0.02
    g = pf.UniformGrid2D(n, n, p, p, -(n - 1) * p / 2, -(n - 1) * p / 2, 0.0)
    sl = _rand_slices(rng, pf.UniformRelay(g), n_freq=n_freq, n_ill=1)
    pts = rng.uniform(-0.6, 0.6, size=(3000, 2))
    ev = pf.ExplicitVoxels((pf.VoxelPlane(0.6, pf.PointList(pts[:1500])),
                            pf.VoxelPlane(0.9, pf.PointList(pts[1500:]))))
    from paper_2501_05244_b200.reconstruct import clear_engine_cache
    clear_engine_cache()
    fused = pf.nursd2(sl, ev).field
    monkeypatch.setattr(A, "_READOUT_FUSED", False)
    clear_engine_cache()
    per_f = pf.nursd2(sl, ev).field
    clear_engine_cache()
    assert O.rel_l2(fused, per_f) < 1e-6
    assert O.rel_l2(fused, O.nursd2(sl, ev)) < 2e-6


def test_config2_composed_small(rng, window):
    """Config-2 family (non-planar relay -> arbitrary voxels) against the composed oracle."""
    from paper_2501_05244_b200.algorithms import nursd3d_explicit
    xy = rng.uniform(-0.3, 0.3, size=(600, 2))
    zz = 0.03 * np.sin(2 * np.pi * xy[:, 0] / 0.6) * np.cos(2 * np.pi * xy[:, 1] / 0.9)
    relay = pf.NonPlanarRelay(pf.PointList(np.column_stack([xy, zz])))
    freqs = 2 * np.pi * 299792458.0 / 0.06 * (1.0 + 0.03 * np.arange(2))
    coeff = rng.normal(size=(1, 600, 2)) + 1j * rng.normal(size=(1, 600, 2))
    sl = pf.FrequencySlices(freqs, coeff, relay, pf.PointList(np.array([[0.0, 0.0, 0.0]])))
    p = 0.6 / 24
    lattice = pf.CuboidGrid(pf.UniformGrid3D(24, 24, 1, p, p, 0.1, -0.3 + p / 2, -0.3 + p / 2, 0.6))
    planes = tuple(pf.VoxelPlane(z, pf.PointList(rng.uniform(-0.15, 0.15, size=(40, 2))))
                   for z in (0.5, 0.7))
    ev = pf.ExplicitVoxels(planes)
    vol = nursd3d_explicit(sl, ev, lattice)
    ref = O.nursd3d_explicit(sl, ev, lattice)
    assert O.rel_l2(vol.field, ref) < TOL


@pytest.mark.parametrize("scatter", ["trilinear", "nearest"])
def test_rsd3d_random_relay_vs_oracle(rng, scatter):
    """rsd3d (reconstruct.py:662-719) on a random curved 3D relay with duplicate lattice
    targets, several frequencies and a time-resolved volume, against the float64 oracle."""
    xy = rng.uniform(-0.3, 0.3, size=(400, 2))
    z = 0.02 * np.sin(2 * np.pi * xy[:, 0] / 0.4) * np.cos(2 * np.pi * xy[:, 1] / 0.5)
    relay = pf.NonPlanarRelay(pf.PointList(np.column_stack([xy, z])))
    F = 3
    freqs = 2 * np.pi * 3e8 / 0.06 * (1 + 0.03 * np.arange(F))
    coeff = rng.normal(size=(1, 400, F)) + 1j * rng.normal(size=(1, 400, F))
    sl = pf.FrequencySlices(freqs, coeff, relay, pf.PointList(np.zeros((1, 3))))
    grid = pf.CuboidGrid(pf.UniformGrid3D(24, 20, 3, 0.025, 0.025, 0.1, -0.29, -0.24, 0.6))
    times = np.array([0.0, 2e-10])
    vol = pf.reconstruct(sl, grid, "rsd3d", scatter=scatter, times=times)
    ref = O.rsd3d(sl, grid, scatter=scatter, times=times)
    assert O.rel_l2(vol.field, ref) < TOL


@pytest.mark.parametrize("stage1,video", [("nursd3d", False), ("rsd3d", False), ("nursd3d", True)])
def test_3d_relay_plus_srsd_vs_composed_oracle(rng, stage1, video):
    """The paper's "3D RSD / 3D NURSD + SRSD": stage 1 of the 3D
    algorithms to the virtual plane, then srsd onto a depth-widening frustum; against the
    composed oracle (reference stage 1 + reference srsd)."""
    xy = rng.uniform(-0.3, 0.3, size=(500, 2))
    zz = 0.03 * np.sin(2 * np.pi * xy[:, 0] / 0.6) * np.cos(2 * np.pi * xy[:, 1] / 0.9)
    relay = pf.NonPlanarRelay(pf.PointList(np.column_stack([xy, zz])))
    F = 3
    freqs = 2 * np.pi * 299792458.0 / 0.06 * (1.0 + 0.03 * np.arange(F))
    coeff = rng.normal(size=(1, 500, F)) + 1j * rng.normal(size=(1, 500, F))
    sl = pf.FrequencySlices(freqs, coeff, relay, pf.PointList(np.array([[0.0, 0.0, 0.0]])))
    n, p = 24, 0.6 / 24
    base = pf.UniformGrid2D(n, n, p, p, -0.3 + p / 2, -0.3 + p / 2, 0.0)
    zs = np.linspace(0.5, 1.1, 4)
    frustum = pf.FrustumGrid(base, zs, zs[0] / zs, zs[0] / zs)
    times = np.array([0.0, 2e-10]) if video else None
    fn = pf.nursd3d_srsd if stage1 == "nursd3d" else pf.rsd3d_srsd
    vol = fn(sl, frustum, times=times)
    ref = O.lattice_srsd(sl, frustum, stage1=stage1, times=times)
    assert O.rel_l2(vol.field, ref) < TOL


@pytest.mark.parametrize("video", [False, True])
def test_nursd2_voxels_arbitrary_depths_vs_per_voxel_planes(rng, video):
    """Voxels at arbitrary depths (VoxelCloud, z-Chebyshev readout) = the reference's nursd2
    on one plane per voxel (reconstruct.py:413-459)."""
    n = 24
    p = 0.02
    g = pf.UniformGrid2D(n, n, p, p, -(n - 1) * p / 2, -(n - 1) * p / 2, 0.0)
    sl = _rand_slices(rng, pf.UniformRelay(g), n_freq=3, n_ill=1)
    pts = np.column_stack([rng.uniform(-0.2, 0.2, size=(150, 2)), rng.uniform(0.5, 1.3, 150)])
    cloud = pf.VoxelCloud(pts)
    times = np.array([0.0, 1.5e-10]) if video else None
    vol = pf.nursd2_voxels(sl, cloud, times=times)
    ref = O.nursd2(sl, cloud.as_explicit(), times=times)
    assert O.rel_l2(vol.field, ref) < TOL


def test_config2_family_voxel_cloud_vs_composed_oracle(rng):
    """Non-planar relay -> voxels at arbitrary depths (config 7 family): nursd3d stage 1 +
    the z-Chebyshev nursd2 readout against the composed oracle with one plane per voxel."""
    from paper_2501_05244_b200.algorithms import nursd3d_explicit
    xy = rng.uniform(-0.3, 0.3, size=(500, 2))
    zz = 0.03 * np.sin(2 * np.pi * xy[:, 0] / 0.6) * np.cos(2 * np.pi * xy[:, 1] / 0.9)
    relay = pf.NonPlanarRelay(pf.PointList(np.column_stack([xy, zz])))
    freqs = 2 * np.pi * 299792458.0 / 0.06 * (1.0 + 0.03 * np.arange(2))
    coeff = rng.normal(size=(1, 500, 2)) + 1j * rng.normal(size=(1, 500, 2))
    sl = pf.FrequencySlices(freqs, coeff, relay, pf.PointList(np.array([[0.0, 0.0, 0.0]])))
    p = 0.6 / 24
    lattice = pf.CuboidGrid(pf.UniformGrid3D(24, 24, 1, p, p, 0.1, -0.3 + p / 2, -0.3 + p / 2, 0.6))
    pts = np.column_stack([rng.uniform(-0.15, 0.15, size=(120, 2)), rng.uniform(0.5, 0.9, 120)])
    cloud = pf.VoxelCloud(pts)
    vol = nursd3d_explicit(sl, cloud, lattice)
    ref = O.nursd3d_explicit(sl, cloud.as_explicit(), lattice)
    assert O.rel_l2(vol.field, ref) < TOL
