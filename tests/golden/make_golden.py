"""Generate golden vectors by running the REFERENCE package (build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

The reference (pure Python, /root/reference/pkg) is imported read-only and run
on small seeded cases; inputs and outputs are written to ``tests/golden/*.npz``.
The GPU box has no /root/reference, so the tests there only read these files.
Nothing here is product code.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import phasorfield as pf                       # noqa: E402
from phasorfield import oracle as pfo          # noqa: E402
from phasorfield import spectral as sp         # noqa: E402
from phasorfield.core import UniformGrid3D     # noqa: E402

R = sys.modules["phasorfield.reconstruct"]     # the package rebinds the name
OUT = os.path.dirname(os.path.abspath(__file__))


def _relay_dict(relay, prefix="relay"):
    d = {f"{prefix}_kind": np.array(relay.kind)}
    if relay.kind == "uniform":
        g = relay.grid
        d[f"{prefix}_grid"] = np.array([g.nx, g.ny, g.dx, g.dy, g.x0, g.y0, g.z], dtype=np.float64)
    elif relay.kind == "nonuniform_planar":
        d[f"{prefix}_points"] = np.asarray(relay.points.points)
        d[f"{prefix}_z"] = np.array(relay.z)
    else:
        d[f"{prefix}_points"] = np.asarray(relay.points.points)
    return d


def _grid_dict(grid):
    d = {"grid_kind": np.array(grid.kind)}
    if grid.kind == "cuboid":
        g = grid.grid
        d["grid_cuboid"] = np.array([g.nx, g.ny, g.nz, g.dx, g.dy, g.dz, g.x0, g.y0, g.z0])
    elif grid.kind == "frustum":
        b = grid.base
        d["grid_base"] = np.array([b.nx, b.ny, b.dx, b.dy, b.x0, b.y0, b.z], dtype=np.float64)
        d["grid_zs"] = np.asarray(grid.zs)
        d["grid_alphas"] = np.asarray(grid.alphas)
        d["grid_betas"] = np.asarray(grid.betas)
    else:
        d["grid_plane_z"] = np.array([p.z for p in grid.planes])
        d["grid_plane_n"] = np.array([p.points.count for p in grid.planes])
        d["grid_points"] = np.vstack([np.asarray(p.points.points) for p in grid.planes])
    return d


def _slices_dict(sl):
    d = {"frequencies": np.asarray(sl.frequencies),
         "coefficients": np.asarray(sl.coefficients),
         "illuminations": np.asarray(sl.illuminations.points)}
    d.update(_relay_dict(sl.relay))
    return d


def centered_relay(n, pitch, z=0.0):
    o = -(n - 1) * pitch / 2.0
    return pf.UniformRelay(pf.UniformGrid2D(n, n, pitch, pitch, o, o, z))


def make_slices(scene, relay, ill, lambda_c=0.06, delta_t=16e-12, n_bins=1024, t0=0.0):
    m = pf.simulate(scene, relay, ill, delta_t=delta_t, n_bins=n_bins, t0=t0)
    return pf.to_frequency(m, pf.build_kernel(lambda_c, n_bins, delta_t))


def two_scatterer(relay, ill=None, **kw):
    scene = pf.Scene((pf.Scatterer((0.03, -0.02, 0.9), 1.0),
                      pf.Scatterer((-0.05, 0.04, 1.0), 0.7)))
    ill = ill if ill is not None else pf.PointList(np.array([[0.0, 0.0], [0.05, -0.03]]))
    return make_slices(scene, relay, ill, **kw)


def save(name, **arrays):
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **arrays)
    print("wrote", name, sum(a.nbytes for a in arrays.values()), "bytes")


def gen_kernel_and_transform():
    rng = np.random.default_rng(20260825)
    kats = []
    for args in [(0.04, 4096, 16e-12), (0.06, 2048, 8e-12), (0.06, 4096, 4e-12),
                 (0.08, 4096, 8e-12), (0.03, 4096, 4e-12), (0.06, 1024, 16e-12),
                 (0.08, 128, 32e-12), (0.06, 512, 16e-12)]:
        k = pf.build_kernel(*args)
        kats.append((args, k.bin_indices, k.frequencies, k.weights))
    d = {}
    for i, (args, b, f, w) in enumerate(kats):
        d[f"k{i}_args"] = np.array(args)
        d[f"k{i}_bins"] = b
        d[f"k{i}_freqs"] = f
        d[f"k{i}_weights"] = w
    # to_frequency on random histograms, several time-axis lengths
    for i, (nb, dt, t0, lam) in enumerate([(128, 32e-12, 1e-10, 0.08), (512, 16e-12, 3e-10, 0.06),
                                           (2048, 8e-12, 0.0, 0.06), (1000, 16e-12, 2e-10, 0.06)]):
        h = rng.uniform(0.0, 5.0, size=(2, 12, nb)).astype(np.float32)
        relay = centered_relay(2, 0.1)
        relay = pf.NonUniformPlanarRelay(pf.PointList(rng.uniform(-1, 1, (12, 2))), 0.0)
        ill = pf.PointList(np.zeros((2, 2)))
        m = pf.TransientMeasurement(relay, ill, h.astype(np.float64), dt, t0=t0)
        k = pf.build_kernel(lam, nb, dt)
        sl = pf.to_frequency(m, k)
        d[f"tf{i}_hist"] = h
        d[f"tf{i}_args"] = np.array([nb, dt, t0, lam])
        d[f"tf{i}_coeff"] = np.asarray(sl.coefficients)
    d["n_kats"] = np.array(len(kats))
    d["n_tf"] = np.array(4)
    save("phasor", **d)


def gen_spectral():
    rng = np.random.default_rng(301)
    d = {}
    shapes = [(6, 10), (8, 8), (9, 7), (15, 15), (16, 12), (21, 28), (22, 11), (64, 64), (140, 140)]
    for i, s in enumerate(shapes):
        u = rng.normal(size=s) + 1j * rng.normal(size=s)
        d[f"c{i}_u"] = u
        d[f"c{i}_fwd"] = sp.cfft_2d(u)
        d[f"c{i}_inv"] = sp.cifft_2d(u)
    d["n_c"] = np.array(len(shapes))
    cases = [(7, 0.45, 3), (16, 0.9, 8), (31, -0.7, 0), (32, 1.3, 31), (33, 1.0, 0), (64, 0.25, 32),
             (140, 0.6, 70), (512, 0.3, 256)]
    for i, (m, a, o) in enumerate(cases):
        u = rng.normal(size=m) + 1j * rng.normal(size=m)
        d[f"s{i}_u"] = u
        d[f"s{i}_args"] = np.array([m, a, o])
        d[f"s{i}_out"] = sp.sfft_1d(u, a, o)
        d[f"s{i}_slow"] = pfo.scaled_dft(u, a, o)
    d["n_s"] = np.array(len(cases))
    u2 = rng.normal(size=(12, 16)) + 1j * rng.normal(size=(12, 16))
    d["s2d_u"] = u2
    d["s2d_out"] = sp.sfft_2d_centered(u2, 0.45, 0.8)
    nu = [((24,), 1e-4), ((12, 10), 1e-8), ((6, 5, 4), 1e-12), ((12, 10), 1e-6),
          ((140, 140), 1e-6), ((9, 7), 1e-12), ((20, 16, 8), 1e-6)]
    for i, (modes, eps) in enumerate(nu):
        n_pts = 300 if len(modes) > 1 and max(modes) > 50 else 50
        pts = rng.uniform(-np.pi, np.pi, size=(n_pts, len(modes)))
        pts[pts >= np.pi] -= 2 * np.pi
        vals = rng.normal(size=n_pts) + 1j * rng.normal(size=n_pts)
        coeff = rng.normal(size=modes) + 1j * rng.normal(size=modes)
        d[f"n{i}_pts"] = pts
        d[f"n{i}_vals"] = vals
        d[f"n{i}_coeff"] = coeff
        d[f"n{i}_modes"] = np.array(modes)
        d[f"n{i}_eps"] = np.array(eps)
        d[f"n{i}_t1"] = sp.nufft1(pts, vals, modes, eps)
        d[f"n{i}_t2"] = sp.nufft2(coeff, pts, eps)
        d[f"n{i}_d1"] = pfo.nudft1(pts, vals, modes)
        d[f"n{i}_d2"] = pfo.nudft2(coeff, pts)
    d["n_n"] = np.array(len(nu))
    save("spectral", **d)


def gen_reconstruct():
    """Reference reconstructions on the reference test suite's own fixtures."""
    relay16 = centered_relay(16, 0.02)
    sl16 = two_scatterer(relay16)
    grid_small = pf.CuboidGrid(UniformGrid3D(4, 3, 2, 0.02, 0.02, 0.1, -0.03, -0.01, 0.85))
    cases = {}

    def put(name, sl, grid, field, **extra):
        d = _slices_dict(sl)
        d.update(_grid_dict(grid))
        d["field"] = np.asarray(field)
        for k, v in extra.items():
            d[k] = np.asarray(v)
        cases[name] = d

    put("rsd_small", sl16, grid_small, R.rsd(sl16, grid_small).field,
        literal=pfo_literal(sl16, grid_small.coordinates()))
    put("rsd_small_noill", sl16, grid_small,
        R.rsd(sl16, grid_small, include_illumination=False).field)
    full16 = pf.CuboidGrid(UniformGrid3D(16, 16, 3, 0.02, 0.02, 0.07, -0.15, -0.15, 0.8))
    put("rsd_full16", sl16, full16, R.rsd(sl16, full16).field)
    put("rsd_none16", sl16, full16, R.rsd(sl16, full16, padding="none").field)
    times = np.array([0.0, 1.0e-9, -2.5e-10])
    put("rsd_video", sl16, grid_small, R.rsd(sl16, grid_small, times=times).field, times=times)

    # the reference's degeneracy-chain fixture (test_reconstruct.py:69-95)
    relay8 = centered_relay(8, 0.02)
    xy = relay8.coordinates()[:, :2]
    rel_p = pf.NonUniformPlanarRelay(pf.PointList(xy), z=0.0)
    rel_3 = pf.NonPlanarRelay(pf.PointList(np.column_stack([xy, np.zeros(len(xy))])))
    ill2 = pf.PointList(np.array([[0.0, 0.0], [0.05, -0.03]]))
    ill3 = pf.PointList(np.array([[0.0, 0.0, 0.0], [0.05, -0.03, 0.0]]))
    sl_u = two_scatterer(relay8)
    sl_p = two_scatterer(rel_p, ill2)
    sl_3 = two_scatterer(rel_3, ill3)
    cgrid = pf.CuboidGrid(UniformGrid3D(8, 8, 2, 0.02, 0.02, 0.08, -0.07, -0.07, 0.86))
    put("chain_rsd", sl_u, cgrid, R.rsd(sl_u, cgrid).field)
    base = relay8.grid
    fr1 = pf.FrustumGrid(base, np.array([0.86, 0.94]), np.ones(2), np.ones(2))
    put("chain_srsd_unit", sl_u, fr1, R.srsd(sl_u, fr1).field)
    fr8 = pf.FrustumGrid(base, np.array([0.86, 0.94]), np.full(2, 0.8), np.full(2, 0.8))
    put("chain_srsd_08", sl_u, fr8, R.srsd(sl_u, fr8).field)
    put("chain_nursd1", sl_p, cgrid, R.nursd1(sl_p, cgrid, eps=1e-8).field)
    planes = tuple(pf.VoxelPlane(z, pf.PointList(xy)) for z in (0.86, 0.94))
    ev = pf.ExplicitVoxels(planes)
    put("chain_nursd2", sl_u, ev, R.nursd2(sl_u, ev, eps=1e-8).field)
    put("chain_nursd3", sl_p, ev, R.nursd3(sl_p, ev, eps=1e-8, lattice_pitch=0.02).field)
    put("chain_hybrid", sl_u, ev, R.srsd_nursd2(sl_u, ev, alpha=1.0, eps=1e-8).field)
    put("chain_nursd3d_flat", sl_3, cgrid, R.nursd3d(sl_3, cgrid, eps=1e-8).field)

    # off-lattice / non-degenerate cases where pad sizes matter
    rng = np.random.default_rng(401)
    pts = rng.uniform(-0.08, 0.08, size=(40, 2))
    rel_r = pf.NonUniformPlanarRelay(pf.PointList(pts), z=0.0)
    sl_r = two_scatterer(rel_r, pf.PointList(np.array([[0.0, 0.0]])))
    g10 = pf.CuboidGrid(UniformGrid3D(10, 9, 3, 0.02, 0.02, 0.06, -0.09, -0.08, 0.85))
    put("nursd1_random", sl_r, g10, R.nursd1(sl_r, g10, eps=1e-6).field)
    vox = tuple(pf.VoxelPlane(z, pf.PointList(rng.uniform(-0.09, 0.09, size=(25, 2))))
                for z in (0.88, 0.95, 1.02))
    evr = pf.ExplicitVoxels(vox)
    put("nursd2_random", sl16, evr, R.nursd2(sl16, evr, eps=1e-6).field)
    put("nursd3_random", sl_r, evr, R.nursd3(sl_r, evr, eps=1e-6).field)
    put("hybrid_random", sl16, evr, R.srsd_nursd2(sl16, evr, alpha=0.7, beta=0.55, eps=1e-6).field)
    frl = pf.FrustumGrid.linear(relay16.grid, np.array([0.85, 0.95, 1.05]), 0.5)
    put("srsd_linear16", sl16, frl, R.srsd(sl16, frl).field)
    frv = pf.FrustumGrid(relay16.grid, np.array([0.9]), np.array([0.6]), np.array([0.45]))
    put("srsd_aniso16", sl16, frv, R.srsd(sl16, frv).field,
        video=R.srsd(sl16, frv, times=np.array([0.0, 5e-10])).field)
    # non-planar relay (config-2 family, small)
    xy3 = rng.uniform(-0.08, 0.08, size=(48, 2))
    zz3 = 0.01 * np.sin(2 * np.pi * xy3[:, 0] / 0.16) * np.cos(2 * np.pi * xy3[:, 1] / 0.24)
    rel_c = pf.NonPlanarRelay(pf.PointList(np.column_stack([xy3, zz3])))
    sl_c = two_scatterer(rel_c, pf.PointList(np.array([[0.0, 0.0, 0.0]])))
    g3 = pf.CuboidGrid(UniformGrid3D(8, 8, 2, 0.02, 0.02, 0.08, -0.07, -0.07, 0.86))
    put("nursd3d_curved", sl_c, g3, R.nursd3d(sl_c, g3, eps=1e-6).field)
    put("rsd3d_curved_tri", sl_c, g3, R.rsd3d(sl_c, g3, scatter="trilinear").field)
    put("rsd3d_curved_near", sl_c, g3, R.rsd3d(sl_c, g3, scatter="nearest").field)
    # odd relay size (odd pads, centred-index shifts)
    relay9 = pf.UniformRelay(pf.UniformGrid2D(9, 7, 0.02, 0.025, -0.08, -0.075, 0.0))
    sl9 = two_scatterer(relay9)
    g9 = pf.CuboidGrid(UniformGrid3D(5, 4, 2, 0.02, 0.025, 0.1, -0.06, -0.05, 0.9))
    put("rsd_odd", sl9, g9, R.rsd(sl9, g9).field)
    put("rsd_odd_none", sl9, pf.CuboidGrid(UniformGrid3D(9, 7, 2, 0.02, 0.025, 0.1, -0.08,
                                                          -0.075, 0.9)),
        R.rsd(sl9, pf.CuboidGrid(UniformGrid3D(9, 7, 2, 0.02, 0.025, 0.1, -0.08, -0.075, 0.9)),
              padding="none").field)
    for name, d in cases.items():
        save(f"rec_{name}", **d)


def pfo_literal(sl, voxels):
    sys.path.insert(0, "/root/reference/pkg/tests")
    from helpers import literal_field
    return literal_field(sl, voxels)


def gen_containers():
    """NLS1 files written by the reference writers (core.py:676-806): every relay
    kind and every volume grid kind, static and time-resolved."""
    from phasorfield import core as C
    rng = np.random.default_rng(707)
    d = os.path.join(OUT, "nls1")
    os.makedirs(d, exist_ok=True)
    ill = pf.PointList(np.array([[0.0, 0.0], [0.1, -0.05]]))
    relays = {
        "uniform": pf.UniformRelay(pf.UniformGrid2D(4, 3, 0.02, 0.025, -0.03, -0.025, 0.0)),
        "planar": pf.NonUniformPlanarRelay(pf.PointList(rng.uniform(-0.1, 0.1, (5, 2))), 0.01),
        "nonplanar": pf.NonPlanarRelay(pf.PointList(rng.uniform(-0.1, 0.1, (6, 3)))),
    }
    for name, relay in relays.items():
        hist = rng.poisson(3.0, size=(2, relay.count, 8)).astype(np.float64)
        m = C.TransientMeasurement(relay, ill, hist, 4e-12, 1.5e-9)
        C.write_dataset(m, os.path.join(d, f"dataset_{name}.nls1"))
    cub = pf.CuboidGrid(UniformGrid3D(3, 2, 2, 0.02, 0.025, 0.1, -0.02, -0.0125, 0.5))
    fru = pf.FrustumGrid(pf.UniformGrid2D(3, 2, 0.02, 0.025, -0.02, -0.0125, 0.0),
                         np.array([0.5, 0.7]), np.array([1.0, 0.7]), np.array([1.0, 0.6]))
    exp = pf.ExplicitVoxels((pf.VoxelPlane(0.5, pf.PointList(rng.uniform(-0.1, 0.1, (3, 2)))),
                             pf.VoxelPlane(0.8, pf.PointList(rng.uniform(-0.1, 0.1, (2, 2))))))
    for name, grid in (("cuboid", cub), ("frustum", fru), ("explicit", exp)):
        f = rng.normal(size=grid.count) + 1j * rng.normal(size=grid.count)
        C.write_volume(C.ReconstructionVolume(grid, f), os.path.join(d, f"volume_{name}.nls1"))
    times = np.array([0.0, 1e-10, 2.5e-10])
    fv = rng.normal(size=(3, cub.count)) + 1j * rng.normal(size=(3, cub.count))
    C.write_volume(C.ReconstructionVolume(cub, fv, times), os.path.join(d, "volume_video.nls1"))


def gen_acceptance():
    """The reference acceptance suite's 20 oracle-consistency scenes (test_acceptance.py:
    204-266, seeds 6000+i): every algorithm path, one or two illuminations, one or two
    scatterers.  Stores the slices, grid, the reference reconstruction and the reference
    oracle.backproject field (the suite's NCC floor: 0.95, 0.9 for the 3D relays)."""
    from phasorfield import sim as S
    names = list(pf.ALGORITHM_NAMES)
    out = {}
    for i in range(20):
        rng = np.random.default_rng(6000 + i)
        algo = names[i % len(names)]
        lambda_c = (0.04, 0.05, 0.06)[i % 3]
        z_mid = float(rng.uniform(1.0, 1.2))
        scat = [S.Scatterer((float(rng.uniform(-0.06, 0.06)), float(rng.uniform(-0.06, 0.06)),
                             z_mid + float(rng.uniform(-0.05, 0.05))), float(rng.uniform(0.6, 1.0)))
                for _ in range(1 + i % 2)]
        scene = S.Scene(tuple(scat))
        side, pitch = 16, 0.02
        g2 = pf.UniformGrid2D(side, side, pitch, pitch, -(side - 1) * pitch / 2,
                              -(side - 1) * pitch / 2, 0.0)
        inner = pf.UniformGrid2D(12, 12, pitch, pitch, -11 * pitch / 2, -11 * pitch / 2, 0.0)
        xy = np.column_stack([c.ravel() for c in np.meshgrid(g2.x_coords(), g2.y_coords())])
        n_ill = 1 + i % 2
        ill_xy = rng.uniform(-0.08, 0.08, size=(n_ill, 2))
        if algo in ("rsd", "srsd", "nursd2", "srsd-nursd2"):
            relay, ill = pf.UniformRelay(g2), pf.PointList(ill_xy)
        elif algo in ("nursd1", "nursd3"):
            jit = rng.uniform(-0.006, 0.006, size=xy.shape)
            relay, ill = pf.NonUniformPlanarRelay(pf.PointList(xy + jit), z=0.0), pf.PointList(ill_xy)
        else:
            zs = rng.uniform(0.0, 0.01, size=len(xy))
            relay = pf.NonPlanarRelay(pf.PointList(np.column_stack([xy, zs])))
            ill = pf.PointList(np.column_stack([ill_xy, np.zeros(n_ill)]))
        sl = make_slices(scene, relay, ill, lambda_c=lambda_c, delta_t=32e-12, n_bins=512)
        z0 = z_mid - 0.09
        if algo in ("rsd", "rsd3d", "nursd3d", "nursd1"):
            grid = pf.CuboidGrid(UniformGrid3D(12, 12, 4, pitch, pitch, 0.06, inner.x0, inner.y0, z0))
        elif algo == "srsd":
            grid = pf.FrustumGrid(g2, z0 + 0.06 * np.arange(4), np.linspace(1.0, 0.85, 4),
                                  np.linspace(1.0, 0.85, 4))
        else:
            planes = [pf.VoxelPlane(z0 + 0.07 * k, pf.PointList(rng.uniform(-0.1, 0.1, size=(120, 2))))
                      for k in range(3)]
            grid = pf.ExplicitVoxels(tuple(planes))
        opts = {"alpha": 0.8} if algo == "srsd-nursd2" else {}
        d = _slices_dict(sl)
        d.update(_grid_dict(grid))
        d["algo"] = np.array(algo)
        d["alpha"] = np.array(opts.get("alpha", np.nan))
        d["field"] = np.asarray(pf.reconstruct(sl, grid, algo, **opts).field)
        d["backproject"] = np.asarray(pfo.backproject(sl, grid.coordinates()))
        d["floor"] = np.array(0.9 if algo in ("rsd3d", "nursd3d") else 0.95)
        out[f"acc{i}"] = d
    for name, d in out.items():
        save(f"acc_{name[3:]}", **d)


def gen_sim():
    """Reference simulator (sim.py:67-129) on small scenes: non-confocal with ambient,
    confocal, no falloff, and a seeded Poisson draw."""
    from phasorfield import sim as S
    relay = pf.UniformRelay(pf.UniformGrid2D(5, 4, 0.05, 0.06, -0.1, -0.09, 0.0))
    ill = pf.PointList(np.array([[0.0, 0.0], [0.05, -0.03]]))
    scene = S.Scene((S.Scatterer((0.02, -0.01, 0.5), 1.0), S.Scatterer((-0.05, 0.04, 0.7), 0.6),
                     S.Scatterer((0.0, 0.0, 0.9), 0.8)), ambient=0.01)
    out = {}
    m = S.simulate(scene, relay, ill, 16e-12, 512, t0=2.5e-9)
    out["hist"] = m.histograms
    out["hist_confocal"] = S.simulate(scene, relay, None, 16e-12, 512, t0=2.5e-9,
                                      confocal=True).histograms
    out["hist_nofalloff"] = S.simulate(scene, relay, ill, 16e-12, 512, t0=2.5e-9,
                                       falloff=False).histograms
    out["hist_poisson"] = S.add_poisson_noise(m, 50.0, seed=7).histograms
    out["scatterers"] = np.array([list(s.position) + [s.albedo] for s in scene.scatterers])
    save("sim", **out)


if __name__ == "__main__":
    gen_acceptance()
    gen_sim()
    gen_kernel_and_transform()
    gen_spectral()
    gen_reconstruct()
    gen_containers()
