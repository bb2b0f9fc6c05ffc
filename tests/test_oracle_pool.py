"""The process-parallel oracle used by the full-size parity tests reproduces the unsplit
oracle bit for bit (plane blocks: per-plane work is independent; frequency terms: added
in ascending order like the reference's _reduce, reconstruct.py:163-168)."""

import numpy as np

import paper_2501_05244_b200 as pf
from oracle import pf_oracle as O
from oracle.pool import oracle_freq_terms, oracle_planes


def _uniform_slices(rng, n=12, F=3):
    p = 0.05
    g = pf.UniformGrid2D(n, n, p, p, -(n - 1) * p / 2, -(n - 1) * p / 2, 0.0)
    freqs = 2 * np.pi * 3e8 / 0.06 * (1 + 0.04 * np.arange(F))
    c = rng.normal(size=(1, n * n, F)) + 1j * rng.normal(size=(1, n * n, F))
    return pf.FrequencySlices(freqs, c, pf.UniformRelay(g), pf.PointList(np.zeros((1, 2)))), g


def test_plane_blocks_equal_unsplit_rsd(rng):
    sl, g = _uniform_slices(rng)
    grid = pf.CuboidGrid(pf.UniformGrid3D(g.nx, g.ny, 7, g.dx, g.dy, 0.1, g.x0, g.y0, 0.4))
    full = O.rsd(sl, grid)
    split = oracle_planes("rsd", sl, grid, 7, procs=3)
    assert np.array_equal(full, split)


def test_plane_blocks_equal_unsplit_srsd(rng):
    sl, g = _uniform_slices(rng, n=8)
    zs = np.linspace(0.5, 1.5, 5)
    grid = pf.FrustumGrid(g, zs, zs[0] / zs, zs[0] / zs)
    assert np.array_equal(O.srsd(sl, grid), oracle_planes("srsd", sl, grid, 5, procs=2))


def test_frequency_terms_equal_unsplit_composed_oracle(rng):
    xy = rng.uniform(-0.3, 0.3, size=(200, 2))
    zz = 0.03 * np.sin(2 * np.pi * xy[:, 0] / 0.6) * np.cos(2 * np.pi * xy[:, 1] / 0.9)
    relay = pf.NonPlanarRelay(pf.PointList(np.column_stack([xy, zz])))
    F = 3
    freqs = 2 * np.pi * 299792458.0 / 0.06 * (1.0 + 0.03 * np.arange(F))
    coeff = rng.normal(size=(1, 200, F)) + 1j * rng.normal(size=(1, 200, F))
    sl = pf.FrequencySlices(freqs, coeff, relay, pf.PointList(np.array([[0.0, 0.0, 0.0]])))
    p = 0.6 / 16
    lattice = pf.CuboidGrid(pf.UniformGrid3D(16, 16, 1, p, p, 0.1, -0.3 + p / 2, -0.3 + p / 2,
                                             0.6))
    planes = tuple(pf.VoxelPlane(z, pf.PointList(rng.uniform(-0.15, 0.15, size=(20, 2))))
                   for z in (0.5, 0.7))
    ev = pf.ExplicitVoxels(planes)
    full = O.nursd3d_explicit(sl, ev, lattice)
    split = oracle_freq_terms("nursd3d_explicit", sl, (ev, lattice), procs=3,
                              z_pitch=sl.shortest_wavelength / 2.0)
    assert np.array_equal(full, split)
