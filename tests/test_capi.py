"""The whole-algorithm C entry points pf_rsd, pf_srsd, pf_nursd1 and pf_nursd2 (include/pfgpu.h), called the way a reference-side
ctypes binding would call it: host geometry and frequency arrays, device
slices / volume / workspace pointers, the caller's stream.  CPU tests cover the planning
and the reference's validation messages (no device needed); GPU tests compare the result
with the float64 oracle (reference rsd / srsd / nursd1 / nursd2, reconstruct.py:208-459) and with
the Python engine.
"""

import ctypes

import numpy as np
import pytest

import paper_2501_05244_b200 as pf
from oracle import pf_oracle as O
from paper_2501_05244_b200 import _lib
from paper_2501_05244_b200.core import illumination_coordinates

TOL = 1e-4


def rsd_args(slices, grid, padding="exact", times=None, include_illumination=True):
    """pf_rsd_args from reference objects (the binding a maintainer would add); the host
    arrays are returned too so they outlive the call."""
    g, vg = slices.relay.grid, grid.grid
    freqs = np.ascontiguousarray(slices.frequencies, dtype=np.float64)
    ill = np.ascontiguousarray(illumination_coordinates(slices.relay, slices.illuminations),
                               dtype=np.float64)
    t = None if times is None else np.ascontiguousarray(times, dtype=np.float64)
    a = _lib.PfRsdArgs(relay_nx=g.nx, relay_ny=g.ny, relay_dx=g.dx, relay_dy=g.dy,
                       relay_x0=g.x0, relay_y0=g.y0, relay_z=g.z, nx=vg.nx, ny=vg.ny, nz=vg.nz,
                       dx=vg.dx, dy=vg.dy, dz=vg.dz, x0=vg.x0, y0=vg.y0, z0=vg.z0,
                       n_freq=freqs.size, n_illum=ill.shape[0],
                       frequencies=freqs.ctypes.data, ill_xyz=ill.ctypes.data,
                       n_frames=0 if t is None else t.size,
                       times=None if t is None else t.ctypes.data,
                       padding_none=int(padding == "none"),
                       include_illum=int(bool(include_illumination)))
    return a, (freqs, ill, t)


def capi_rsd(slices, grid, **kw):
    import torch
    a, keep = rsd_args(slices, grid, **kw)
    lib = _lib.load()
    nbytes = lib.pf_rsd_workspace_bytes(ctypes.byref(a))
    assert nbytes > 0, _lib.last_error()
    c = np.asarray(slices.coefficients)                       # [I, D, F]
    coeff = torch.from_numpy(np.ascontiguousarray(c.transpose(2, 0, 1)).astype(np.complex64)).cuda()
    frames = max(1, a.n_frames)
    vol = torch.empty((frames, grid.count), dtype=torch.complex64, device="cuda")
    ws = torch.empty((nbytes,), dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    rc = lib.pf_rsd(ctypes.byref(a), coeff.data_ptr(), vol.data_ptr(), ws.data_ptr(), nbytes, s)
    assert rc == 0, _lib.last_error()
    torch.cuda.synchronize()
    return vol.cpu().numpy()


def _scene(rng, n, F=4, n_ill=1, nz=3, off=0, nx=None, ny=None, dz=0.25, spacing=0.02):
    p = 2.0 / n
    g = pf.UniformGrid2D(n, n, p, p, -1 + p / 2, -1 + p / 2, 0.0)
    freqs = 2 * np.pi * 3e8 / 0.06 * (1 + spacing * np.arange(F))
    c = rng.normal(size=(n_ill, n * n, F)) + 1j * rng.normal(size=(n_ill, n * n, F))
    ill = pf.PointList(rng.uniform(-0.3, 0.3, size=(n_ill, 2)))
    sl = pf.FrequencySlices(freqs, c, pf.UniformRelay(g), ill)
    nx, ny = nx or n, ny or n
    grid = pf.CuboidGrid(pf.UniformGrid3D(nx, ny, nz, p, p, dz, g.x0 + off * p, g.y0 + off * p, 0.5))
    return sl, grid


# ---------------------------------------------------------------- CPU: planning + validation

def test_workspace_bytes_config4_geometry():
    from paper_2501_05244_b200 import configs
    cfg = configs.config(4)
    k = configs.kernel(cfg)
    sl = type("S", (), dict(frequencies=k.frequencies, relay=cfg.relay,
                            illuminations=cfg.illuminations))()
    a, _ = rsd_args(sl, cfg.grid)
    nbytes = _lib.load().pf_rsd_workspace_bytes(ctypes.byref(a))
    # Uhat (32 x 1024^2 c64 = 256 MiB) + 3 lanes x 4 planes of A and B workspaces
    assert 256 << 20 < nbytes < 512 << 20


@pytest.mark.parametrize("change,match", [
    (dict(dx=0.05), "pitch"), (dict(x0=0.013), "origin"), (dict(z0=-0.2), "beyond the relay"),
    (dict(nx=20), "padding='none'")])
def test_validation_messages(rng, change, match):
    sl, grid = _scene(rng, 32)
    a, keep = rsd_args(sl, grid, padding="none" if match == "padding='none'" else "exact")
    for k, v in change.items():
        setattr(a, k, v)
    assert _lib.load().pf_rsd_workspace_bytes(ctypes.byref(a)) == -1
    assert match in _lib.last_error()


# ---------------------------------------------------------------- GPU: results

@pytest.mark.gpu
@pytest.mark.parametrize("case", [
    dict(n=64),                                 # P = 128 register path, Horner C
    dict(n=64, F=40),                           # Horner in 32-frequency blocks
    dict(n=64, n_ill=2),                        # two illuminations (per-frequency phases)
    dict(n=40, nx=30, ny=24, off=3),            # generic pad, offset window
    dict(n=128, nz=5),                          # P = 256
])
def test_pf_rsd_matches_oracle_and_engine(rng, case):
    sl, grid = _scene(rng, **case)
    got = capi_rsd(sl, grid)[0]
    ref = O.rsd(sl, grid)
    assert O.rel_l2(got, ref) < TOL
    eng = pf.rsd(sl, grid).field
    assert O.rel_l2(got, eng) < 1e-5


@pytest.mark.gpu
def test_pf_rsd_video_and_no_padding(rng):
    sl, grid = _scene(rng, 32, F=3)
    times = np.array([0.0, 1.5e-10, 4e-10])
    got = capi_rsd(sl, grid, times=times)
    assert O.rel_l2(got, O.rsd(sl, grid, times=times)) < TOL
    got = capi_rsd(sl, grid, padding="none", include_illumination=False)[0]
    assert O.rel_l2(got, O.rsd(sl, grid, padding="none", include_illumination=False)) < TOL


# ---------------------------------------------------------------- pf_srsd

def srsd_args(slices, frustum, times=None, include_illumination=True):
    g = slices.relay.grid
    zs = np.ascontiguousarray(frustum.zs, dtype=np.float64)
    al = np.ascontiguousarray(frustum.alphas, dtype=np.float64)
    be = np.ascontiguousarray(frustum.betas, dtype=np.float64)
    freqs = np.ascontiguousarray(slices.frequencies, dtype=np.float64)
    ill = np.ascontiguousarray(illumination_coordinates(slices.relay, slices.illuminations),
                               dtype=np.float64)
    t = None if times is None else np.ascontiguousarray(times, dtype=np.float64)
    a = _lib.PfSrsdArgs(nx=g.nx, ny=g.ny, relay_dx=g.dx, relay_dy=g.dy, relay_x0=g.x0,
                        relay_y0=g.y0, relay_z=g.z, nz=zs.size, zs=zs.ctypes.data,
                        alphas=al.ctypes.data, betas=be.ctypes.data, n_freq=freqs.size,
                        n_illum=ill.shape[0], frequencies=freqs.ctypes.data,
                        ill_xyz=ill.ctypes.data, n_frames=0 if t is None else t.size,
                        times=None if t is None else t.ctypes.data,
                        include_illum=int(bool(include_illumination)))
    return a, (zs, al, be, freqs, ill, t)


def capi_srsd(slices, frustum, **kw):
    import torch
    a, keep = srsd_args(slices, frustum, **kw)
    lib = _lib.load()
    nbytes = lib.pf_srsd_workspace_bytes(ctypes.byref(a))
    assert nbytes > 0, _lib.last_error()
    c = np.asarray(slices.coefficients)
    coeff = torch.from_numpy(np.ascontiguousarray(c.transpose(2, 0, 1)).astype(np.complex64)).cuda()
    vol = torch.empty((max(1, a.n_frames), frustum.count), dtype=torch.complex64, device="cuda")
    ws = torch.empty((nbytes,), dtype=torch.uint8, device="cuda")
    rc = lib.pf_srsd(ctypes.byref(a), coeff.data_ptr(), vol.data_ptr(), ws.data_ptr(), nbytes,
                     torch.cuda.current_stream().cuda_stream)
    assert rc == 0, _lib.last_error()
    torch.cuda.synchronize()
    return vol.cpu().numpy()


def _frustum(g, nz=4, z0=0.6, z1=1.8):
    zs = np.linspace(z0, z1, nz)
    return pf.FrustumGrid(g, zs, zs[0] / zs, zs[0] / zs)


def test_srsd_workspace_and_validation(rng):
    sl, _ = _scene(rng, 32)
    fr = _frustum(sl.relay.grid)
    a, keep = srsd_args(sl, fr)
    assert _lib.load().pf_srsd_workspace_bytes(ctypes.byref(a)) > 0
    a.relay_z = 1.0                                       # planes no longer beyond the relay
    assert _lib.load().pf_srsd_workspace_bytes(ctypes.byref(a)) == -1
    assert "beyond the relay" in _lib.last_error()


@pytest.mark.gpu
@pytest.mark.parametrize("case", [
    dict(n=32),                 # P = 64 generic Stockham pad, Q = 128
    dict(n=64),                 # P = 128 register path, Q = 256 register Bluestein, Horner C
    dict(n=64, F=40),           # Horner blocks
    dict(n=48, n_ill=2),        # P = 96 generic, two illuminations
    dict(n=128, nz=3),          # P = 256, Q = 512
])
def test_pf_srsd_matches_oracle_and_engine(rng, case):
    nz = case.pop("nz", 4)
    sl, _ = _scene(rng, **case)
    fr = _frustum(sl.relay.grid, nz=nz)
    got = capi_srsd(sl, fr)[0]
    ref = O.srsd(sl, fr)
    assert O.rel_l2(got, ref) < TOL
    assert O.rel_l2(got, pf.srsd(sl, fr).field) < 1e-5


@pytest.mark.gpu
def test_pf_srsd_video(rng):
    sl, _ = _scene(rng, 32, F=3)
    fr = _frustum(sl.relay.grid, nz=3)
    times = np.array([0.0, 2e-10])
    got = capi_srsd(sl, fr, times=times)
    assert O.rel_l2(got, O.srsd(sl, fr, times=times)) < TOL


# ---------------------------------------------------------------- pf_nursd1

def nursd1_args(slices, grid, eps=1e-6, times=None, include_illumination=True):
    vg = grid.grid
    xy = np.ascontiguousarray(np.asarray(slices.relay.points.points)[:, :2], dtype=np.float64)
    freqs = np.ascontiguousarray(slices.frequencies, dtype=np.float64)
    ill = np.ascontiguousarray(illumination_coordinates(slices.relay, slices.illuminations),
                               dtype=np.float64)
    t = None if times is None else np.ascontiguousarray(times, dtype=np.float64)
    a = _lib.PfNursd1Args(n_points=xy.shape[0], relay_xy=xy.ctypes.data, relay_z=slices.relay.z,
                          nx=vg.nx, ny=vg.ny, nz=vg.nz, dx=vg.dx, dy=vg.dy, dz=vg.dz, x0=vg.x0,
                          y0=vg.y0, z0=vg.z0, n_freq=freqs.size, n_illum=ill.shape[0],
                          frequencies=freqs.ctypes.data, ill_xyz=ill.ctypes.data,
                          n_frames=0 if t is None else t.size,
                          times=None if t is None else t.ctypes.data, eps=eps,
                          include_illum=int(bool(include_illumination)))
    return a, (xy, freqs, ill, t)


def capi_nursd1(slices, grid, **kw):
    import torch
    a, keep = nursd1_args(slices, grid, **kw)
    lib = _lib.load()
    nbytes = lib.pf_nursd1_workspace_bytes(ctypes.byref(a))
    assert nbytes > 0, _lib.last_error()
    c = np.asarray(slices.coefficients)
    coeff = torch.from_numpy(np.ascontiguousarray(c.transpose(2, 0, 1)).astype(np.complex64)).cuda()
    vol = torch.empty((max(1, a.n_frames), grid.count), dtype=torch.complex64, device="cuda")
    ws = torch.empty((nbytes,), dtype=torch.uint8, device="cuda")
    rc = lib.pf_nursd1(ctypes.byref(a), coeff.data_ptr(), vol.data_ptr(), ws.data_ptr(), nbytes,
                       torch.cuda.current_stream().cuda_stream)
    assert rc == 0, _lib.last_error()
    torch.cuda.synchronize()
    return vol.cpu().numpy()


def _scatter_scene(rng, n=64, n_pts=2048, F=2, n_ill=1, nz=3, lattice=False):
    p = 2.0 / n
    if lattice:
        g = pf.UniformGrid2D(n, n, p, p, -1 + p / 2, -1 + p / 2, 0.0)
        xy = pf.grid_coordinates(g).points
        xy = xy[rng.random(xy.shape[0]) < 0.5]
    else:
        xy = rng.uniform(-1.0, 1.0, size=(n_pts, 2))
    relay = pf.NonUniformPlanarRelay(pf.PointList(xy), 0.0)
    freqs = 2 * np.pi * 3e8 / 0.06 * (1 + 0.02 * np.arange(F))
    c = rng.normal(size=(n_ill, relay.count, F)) + 1j * rng.normal(size=(n_ill, relay.count, F))
    ill = pf.PointList(rng.uniform(-0.3, 0.3, size=(n_ill, 2)))
    sl = pf.FrequencySlices(freqs, c, relay, ill)
    grid = pf.CuboidGrid(pf.UniformGrid3D(n, n, nz, p, p, 0.3, -1 + p / 2, -1 + p / 2, 0.5))
    return sl, grid


def test_nursd1_workspace_and_validation(rng):
    sl, grid = _scatter_scene(rng)
    a, keep = nursd1_args(sl, grid)
    lib = _lib.load()
    n = lib.pf_nursd1_workspace_bytes(ctypes.byref(a))
    # off-lattice points: the reference pad P = 140, fine grid 280 x 280, F x I = 2
    assert n > 2 * 8 * (280 * 280 + 140 * 140)
    a.eps = 1.0
    assert lib.pf_nursd1_workspace_bytes(ctypes.byref(a)) == -1
    assert "accuracy target" in _lib.last_error()
    a.eps = 1e-6
    a.z0 = -0.5
    assert lib.pf_nursd1_workspace_bytes(ctypes.byref(a)) == -1
    assert "beyond the relay" in _lib.last_error()


@pytest.mark.gpu
@pytest.mark.parametrize("case", [
    dict(),                           # off-lattice: reference pad P = 140, generic path
    dict(n_ill=2, F=3),               # two illuminations
    dict(lattice=True),               # on-lattice: P = 128 register path, pow2 type-1 finish, Horner C
    dict(lattice=True, F=40),         # Horner in 32-frequency blocks
    dict(kw=dict(eps=1e-9)),          # tighter stencil (w = 6; 11 for the Gaussian)
])
def test_pf_nursd1_matches_oracle_and_engine(rng, case):
    kw = case.pop("kw", {})
    sl, grid = _scatter_scene(rng, **case)
    got = capi_nursd1(sl, grid, **kw)[0]
    assert O.rel_l2(got, O.nursd1(sl, grid, **kw)) < TOL
    assert O.rel_l2(got, pf.nursd1(sl, grid, **kw).field) < 1e-5


@pytest.fixture
def gaussian_window(monkeypatch):
    """The reference's Gaussian stencil in both planners (Python plans, C entry points)."""
    from paper_2501_05244_b200 import nufft as nu
    monkeypatch.setattr(nu, "DEFAULT_WINDOW", "gaussian")
    prev = _lib.call("pf_nufft_window", 0)
    yield
    _lib.call("pf_nufft_window", prev)


@pytest.mark.gpu
def test_pf_nursd1_and_nursd2_gaussian_window(rng, gaussian_window):
    """The C planner's Gaussian plan (pf_nufft_window(0)) equals the Python one: the C entry
    points reproduce the engines and the oracle with the reference's own stencil."""
    sl, grid = _scatter_scene(rng)
    got = capi_nursd1(sl, grid)[0]
    assert O.rel_l2(got, O.nursd1(sl, grid)) < 2e-6
    assert O.rel_l2(got, pf.nursd1(sl, grid).field) < 1e-5
    sl, ev = _voxel_scene(rng)
    got = capi_nursd2(sl, ev)[0]
    assert O.rel_l2(got, O.nursd2(sl, ev)) < 2e-6
    assert O.rel_l2(got, pf.nursd2(sl, ev).field) < 1e-5


@pytest.mark.gpu
def test_pf_nursd1_video_without_illumination(rng):
    sl, grid = _scatter_scene(rng, n=32, n_pts=512, F=3)
    times = np.array([0.0, 2e-10])
    got = capi_nursd1(sl, grid, times=times, include_illumination=False)
    ref = O.nursd1(sl, grid, times=times, include_illumination=False)
    assert O.rel_l2(got, ref) < TOL


# ---------------------------------------------------------------- pf_nursd2

def nursd2_args(slices, voxels, eps=1e-6, times=None, include_illumination=True):
    g = slices.relay.grid
    zs = np.ascontiguousarray([p.z for p in voxels.planes], dtype=np.float64)
    cnt = np.ascontiguousarray([p.points.count for p in voxels.planes], dtype=np.int64)
    xy = np.ascontiguousarray(np.vstack([np.asarray(p.points.points) for p in voxels.planes]),
                              dtype=np.float64)
    freqs = np.ascontiguousarray(slices.frequencies, dtype=np.float64)
    ill = np.ascontiguousarray(illumination_coordinates(slices.relay, slices.illuminations),
                               dtype=np.float64)
    t = None if times is None else np.ascontiguousarray(times, dtype=np.float64)
    a = _lib.PfNursd2Args(relay_nx=g.nx, relay_ny=g.ny, relay_dx=g.dx, relay_dy=g.dy,
                          relay_x0=g.x0, relay_y0=g.y0, relay_z=g.z, n_planes=zs.size,
                          plane_z=zs.ctypes.data, plane_count=cnt.ctypes.data,
                          voxel_xy=xy.ctypes.data, n_freq=freqs.size, n_illum=ill.shape[0],
                          frequencies=freqs.ctypes.data, ill_xyz=ill.ctypes.data,
                          n_frames=0 if t is None else t.size,
                          times=None if t is None else t.ctypes.data, eps=eps,
                          include_illum=int(bool(include_illumination)))
    return a, (zs, cnt, xy, freqs, ill, t)


def capi_nursd2(slices, voxels, **kw):
    import torch
    a, keep = nursd2_args(slices, voxels, **kw)
    lib = _lib.load()
    nbytes = lib.pf_nursd2_workspace_bytes(ctypes.byref(a))
    assert nbytes > 0, _lib.last_error()
    c = np.asarray(slices.coefficients)
    coeff = torch.from_numpy(np.ascontiguousarray(c.transpose(2, 0, 1)).astype(np.complex64)).cuda()
    vol = torch.empty((max(1, a.n_frames), voxels.count), dtype=torch.complex64, device="cuda")
    ws = torch.empty((nbytes,), dtype=torch.uint8, device="cuda")
    rc = lib.pf_nursd2(ctypes.byref(a), coeff.data_ptr(), vol.data_ptr(), ws.data_ptr(), nbytes,
                       torch.cuda.current_stream().cuda_stream)
    assert rc == 0, _lib.last_error()
    torch.cuda.synchronize()
    return vol.cpu().numpy()


def _voxel_scene(rng, n=24, F=2, n_ill=1, zs=(0.7, 0.9), per_plane=50):
    p = 0.02
    g = pf.UniformGrid2D(n, n, p, p, -(n - 1) * p / 2, -(n - 1) * p / 2, 0.0)
    freqs = 2 * np.pi * 3e8 / 0.06 * (1 + 0.02 * np.arange(F))
    c = rng.normal(size=(n_ill, n * n, F)) + 1j * rng.normal(size=(n_ill, n * n, F))
    ill = pf.PointList(rng.uniform(-0.1, 0.1, size=(n_ill, 2)))
    sl = pf.FrequencySlices(freqs, c, pf.UniformRelay(g), ill)
    planes = tuple(pf.VoxelPlane(z, pf.PointList(rng.uniform(-0.2, 0.2, size=(per_plane, 2))))
                   for z in zs)
    return sl, pf.ExplicitVoxels(planes)


def test_nursd2_workspace_and_validation(rng):
    sl, ev = _voxel_scene(rng)
    a, keep = nursd2_args(sl, ev)
    lib = _lib.load()
    assert lib.pf_nursd2_workspace_bytes(ctypes.byref(a)) > 0
    a.relay_z = 0.8                                       # plane 0.7 no longer beyond the relay
    assert lib.pf_nursd2_workspace_bytes(ctypes.byref(a)) == -1
    assert "beyond the relay" in _lib.last_error()
    a.relay_z = 0.0
    a.eps = 0.5
    assert lib.pf_nursd2_workspace_bytes(ctypes.byref(a)) == -1
    assert "accuracy target" in _lib.last_error()


@pytest.mark.gpu
@pytest.mark.parametrize("case", [
    dict(),                                       # two planes, one illumination
    dict(n_ill=2, F=3),                           # two illuminations
    dict(zs=(0.5, 0.6, 0.8, 1.1), per_plane=200),
    dict(n=64, zs=(0.9,), per_plane=3000),        # larger pad, one plane
])
def test_pf_nursd2_matches_oracle_and_engine(rng, case):
    sl, ev = _voxel_scene(rng, **case)
    got = capi_nursd2(sl, ev)[0]
    assert O.rel_l2(got, O.nursd2(sl, ev)) < TOL
    assert O.rel_l2(got, pf.nursd2(sl, ev).field) < 1e-5


@pytest.mark.gpu
def test_pf_nursd2_video_without_illumination(rng):
    sl, ev = _voxel_scene(rng, F=3)
    times = np.array([0.0, 2e-10])
    got = capi_nursd2(sl, ev, times=times, include_illumination=False)
    ref = O.nursd2(sl, ev, times=times, include_illumination=False)
    assert O.rel_l2(got, ref) < TOL
