"""GPU parity: K1 temporal transform, FFT core and rsd against the oracle / golden vectors."""

import numpy as np
import pytest
import torch

import paper_2501_05244_b200 as pf
from oracle import pf_oracle as O
from golden_io import grid_from, load, slices_from

pytestmark = pytest.mark.gpu
TOL = 1e-4   # north-star tolerance: relative L2 on the complex volume, fp32 vs float64


def _argmax_same(a, b, shape):
    pa = np.abs(a.reshape(shape)).max(axis=0)
    pb = np.abs(b.reshape(shape)).max(axis=0)
    return int(np.argmax(pa)) == int(np.argmax(pb))


@pytest.mark.parametrize("i", range(4))
def test_to_frequency_golden(i):
    d = load("phasor")
    nb, dt, t0, lam = d[f"tf{i}_args"]
    h = d[f"tf{i}_hist"]
    relay = pf.NonUniformPlanarRelay(pf.PointList(np.zeros((h.shape[1], 2))), 0.0)
    ill = pf.PointList(np.zeros((h.shape[0], 2)))
    m = pf.TransientMeasurement(relay, ill, h, dt, t0=t0)
    k = pf.build_kernel(lam, int(nb), dt)
    sl = pf.to_frequency(m, k)
    assert O.rel_l2(sl.coefficients, d[f"tf{i}_coeff"]) < 1e-6


def test_to_frequency_kats(rng):
    # reference test_phasor.py:94-125: single delta, direct weighted DFT, linearity
    n_bins, dt, t0, b = 512, 16e-12, 3e-10, 41
    relay = pf.NonUniformPlanarRelay(pf.PointList(np.zeros((4, 2))), 0.0)
    ill = pf.PointList(np.zeros((1, 2)))
    h = np.zeros((1, 4, n_bins), np.float32)
    h[0, 2, b] = 2.5
    k = pf.build_kernel(0.06, n_bins, dt)
    sl = pf.to_frequency(pf.TransientMeasurement(relay, ill, h, dt, t0=t0), k)
    pred = k.weights * 2.5 * np.exp(-1j * k.frequencies * (t0 + b * dt))
    assert O.rel_linf(sl.coefficients[0, 2], pred) < 1e-6
    assert np.all(sl.coefficients[0, [0, 1, 3]] == 0)
    h1 = rng.uniform(0, 1, (1, 4, 128)).astype(np.float32)
    h2 = rng.uniform(0, 1, (1, 4, 128)).astype(np.float32)
    k2 = pf.build_kernel(0.08, 128, 32e-12)
    c = [pf.to_frequency(pf.TransientMeasurement(relay, ill, h, 32e-12), k2).coefficients
         for h in (h1, h2, 2 * h1 + 3 * h2)]
    assert O.rel_linf(c[2], 2 * c[0] + 3 * c[1]) < 1e-5


@pytest.mark.parametrize("T", [64, 128, 1024, 2048, 4096, 8192, 960, 1000])
def test_to_frequency_sizes(rng, T):
    dt = 4e-12 if T >= 4096 else 8e-12
    relay = pf.NonUniformPlanarRelay(pf.PointList(np.zeros((37, 2))), 0.0)
    ill = pf.PointList(np.zeros((2, 2)))
    h = rng.poisson(3.0, size=(2, 37, T)).astype(np.float32)
    lam = 40 * dt * 3e8 / 4 if T < 256 else 0.03 * T * dt / (4096 * 4e-12)
    k = pf.build_kernel(max(lam, 0.006), T, dt, threshold=0.001)
    sl = pf.to_frequency(pf.TransientMeasurement(relay, ill, h, dt, t0=2e-10), k)
    ref = O.to_frequency(h, k.bin_indices, k.frequencies, k.weights, 2e-10)
    assert O.rel_l2(sl.coefficients, ref) < 2e-6


@pytest.mark.parametrize("n", [1, 2, 3, 5, 7, 8, 11, 12, 13, 16, 17, 30, 49, 64, 97, 121, 128, 140, 175,
                               194, 280, 350, 512, 525, 700, 1024, 1050, 2048, 2100])
def test_fft_lines_vs_numpy(rng, n):
    from paper_2501_05244_b200 import _device as dev
    x = (rng.normal(size=(3, n)) + 1j * rng.normal(size=(3, n))).astype(np.complex64)
    t = torch.from_numpy(x).cuda()
    dev.fft_lines(t, n, 3, 1, 0, n, 1, -1)
    assert O.rel_l2(t.cpu().numpy(), np.fft.fft(x.astype(np.complex128), axis=1)) < 2e-6
    dev.fft_lines(t, n, 3, 1, 0, n, 1, +1, 1.0 / n)
    assert O.rel_l2(t.cpu().numpy(), x) < 2e-6


@pytest.mark.parametrize("shape", [(6, 10), (9, 7), (64, 64), (140, 140), (20, 16, 8),
                                   (350, 12), (700, 5), (1050, 3), (3, 140, 280), (41, 175)])
def test_fftn_vs_numpy(rng, shape):
    from paper_2501_05244_b200 import _device as dev
    x = (rng.normal(size=(2,) + shape) + 1j * rng.normal(size=(2,) + shape)).astype(np.complex64)
    t = torch.from_numpy(x).cuda()
    dev.fftn_natural(t, shape, 2, -1)
    ref = np.fft.fftn(x.astype(np.complex128), axes=tuple(range(1, len(shape) + 1)))
    assert O.rel_l2(t.cpu().numpy(), ref) < 2e-6


@pytest.mark.parametrize("P,ny,nx,nb", [(128, 64, 64, 3), (128, 37, 50, 2), (256, 128, 128, 1),
                                         (512, 256, 256, 2), (512, 255, 3, 1), (1024, 512, 512, 2),
                                         (1024, 1024, 1000, 1), (128, 1, 1, 1)])
def test_relay_spectra_fast_vs_numpy(rng, P, ny, nx, nb):
    """pf_relay_spectra_fast (register path) = transposed cfft2 of the centred embed
    (reference reconstruct.py:113-119,259-260), natural order, float64 numpy reference."""
    from paper_2501_05244_b200 import _device as dev, _lib
    x = (rng.normal(size=(nb, ny, nx)) + 1j * rng.normal(size=(nb, ny, nx))).astype(np.complex64)
    emb = np.zeros((nb, P, P), np.complex128)
    iy = (np.arange(ny) - ny // 2) % P
    ix = (np.arange(nx) - nx // 2) % P
    emb[:, iy[:, None], ix[None, :]] = x
    ref = np.fft.fft2(emb).transpose(0, 2, 1)
    src = torch.from_numpy(x).cuda()
    out = torch.full((nb, P, P), complex(np.nan, np.nan), dtype=torch.complex64, device="cuda")
    plan = dev.fft_plan(P, src.device)
    _lib.call("pf_relay_spectra_fast", dev.ptr(src), nb, ny, nx, ny * nx, dev.ptr(out), P,
              plan.ref, dev.stream_ptr())
    torch.cuda.synchronize()
    assert O.rel_l2(out.cpu().numpy(), ref) < 2e-6


RSD_CASES = ["rsd_small", "rsd_small_noill", "rsd_full16", "rsd_none16", "rsd_video",
             "chain_rsd", "rsd_odd", "rsd_odd_none"]


@pytest.mark.parametrize("name", RSD_CASES)
def test_rsd_golden(name):
    d = load(f"rec_{name}")
    sl, grid = slices_from(d), grid_from(d)
    kw = {}
    if "noill" in name:
        kw["include_illumination"] = False
    if "none" in name:
        kw["padding"] = "none"
    if name == "rsd_video":
        kw["times"] = d["times"]
    vol = pf.rsd(sl, grid, **kw)
    assert O.rel_l2(vol.field, d["field"]) < TOL
    if "literal" in d:
        assert O.rel_l2(vol.field, d["literal"]) < TOL
    if name != "rsd_video":
        assert _argmax_same(vol.field, d["field"], grid.shape)


def test_rsd_repeat_is_bit_identical():
    d = load("rec_rsd_full16")
    sl, grid = slices_from(d), grid_from(d)
    a = pf.rsd(sl, grid).field
    b = pf.rsd(sl, grid, threads=4).field
    assert np.array_equal(a, b)


def test_rsd_from_device_slices_matches_host_path():
    d = load("rec_chain_rsd")
    sl, grid = slices_from(d), grid_from(d)
    dsl = pf.DeviceFrequencySlices(sl.frequencies,
                                   torch.from_numpy(np.ascontiguousarray(
                                       sl.coefficients.transpose(2, 0, 1)).astype(np.complex64)).cuda(),
                                   sl.relay, sl.illuminations)
    assert np.array_equal(pf.rsd(dsl, grid).field, pf.rsd(sl, grid).field)


def test_rsd_c0_like_end_to_end(rng):
    """A config-0 shaped (smaller) run from transients through rsd, against the oracle."""
    n, T, dt = 32, 2048, 8e-12
    pitch = 2.0 / n
    relay = pf.UniformRelay(pf.UniformGrid2D(n, n, pitch, pitch, -1 + pitch / 2, -1 + pitch / 2, 0.0))
    ill = pf.PointList(np.array([[0.0, 0.0]]))
    h = rng.poisson(0.5, size=(1, n * n, T)).astype(np.float32)
    h[0, :, 700:720] += 20.0
    m = pf.TransientMeasurement(relay, ill, h, dt)
    k = pf.build_kernel(0.06, T, dt)
    sl = pf.to_frequency(m, k)
    grid = pf.CuboidGrid(pf.UniformGrid3D(n, n, 6, pitch, pitch, 0.3, -1 + pitch / 2,
                                          -1 + pitch / 2, 0.5))
    vol = pf.rsd(sl, grid)
    ref = O.rsd(sl.to_host(), grid)
    assert O.rel_l2(vol.field, ref) < TOL
    assert _argmax_same(vol.field, ref, grid.shape)


def _random_slices(rng, relay, n_freq=4, n_ill=1, w0=2 * np.pi * 3e8 / 0.06):
    freqs = w0 * (1.0 + 0.02 * np.arange(n_freq))
    D = relay.count
    coeff = (rng.normal(size=(n_ill, D, n_freq)) + 1j * rng.normal(size=(n_ill, D, n_freq)))
    ill = pf.PointList(rng.uniform(-0.5, 0.5, size=(n_ill, 2)))
    return pf.FrequencySlices(freqs, coeff, relay, ill)


@pytest.mark.parametrize("n,nx,ny,off,n_ill,video", [
    (64, 64, 64, 0, 1, False),      # P = 128 register path, config-0 geometry
    (64, 40, 24, 3, 2, False),      # offset output window, two illuminations (MULTI kernel)
    (128, 128, 128, 0, 1, True),    # P = 256, time-resolved frames
    (256, 256, 256, 0, 1, False),   # P = 512
])
def test_rsd_register_path_vs_oracle(rng, n, nx, ny, off, n_ill, video):
    pitch = 2.0 / n
    g = pf.UniformGrid2D(n, n, pitch, pitch, -1 + pitch / 2, -1 + pitch / 2, 0.0)
    relay = pf.UniformRelay(g)
    sl = _random_slices(rng, relay, n_freq=3, n_ill=n_ill)
    x0 = g.x0 + pitch * ((n - nx) // 2 + off)
    y0 = g.y0 + pitch * ((n - ny) // 2 - off)
    grid = pf.CuboidGrid(pf.UniformGrid3D(nx, ny, 3, pitch, pitch, 0.37, x0, y0, 0.45))
    times = np.array([0.0, 2e-10, -1e-10]) if video else None
    from paper_2501_05244_b200.reconstruct import RsdEngine
    eng = RsdEngine(sl, grid, times=times)
    assert eng.prop.transposed, (eng.px, eng.py)
    vol = pf.rsd(sl, grid, times=times)
    ref = O.rsd(sl, grid, times=times)
    assert O.rel_l2(vol.field, ref) < TOL
    if not video:
        assert _argmax_same(vol.field, ref, grid.shape)


def test_rsd_register_path_literal_subsample(rng):
    """Exact physics (1/r literal sum, reference helpers.py:69-101) on a voxel subsample."""
    n = 64
    pitch = 2.0 / n
    g = pf.UniformGrid2D(n, n, pitch, pitch, -1 + pitch / 2, -1 + pitch / 2, 0.0)
    sl = _random_slices(rng, pf.UniformRelay(g), n_freq=2)
    grid = pf.CuboidGrid(pf.UniformGrid3D(n, n, 2, pitch, pitch, 0.5, g.x0, g.y0, 0.6))
    vol = pf.rsd(sl, grid)
    idx = rng.choice(grid.count, size=40, replace=False)
    lit = O.literal_field(sl, grid.coordinates()[idx])
    assert O.rel_l2(vol.field[idx], lit) < TOL


def test_graphed_run_matches_eager(rng):
    """CUDA-graph replay of the propagation equals the eager launch sequence bitwise."""
    n = 64
    p = 2.0 / n
    g = pf.UniformGrid2D(n, n, p, p, -1 + p / 2, -1 + p / 2, 0.0)
    sl = _random_slices(rng, pf.UniformRelay(g), n_freq=3)
    grid = pf.CuboidGrid(pf.UniformGrid3D(n, n, 5, p, p, 0.3, g.x0, g.y0, 0.5))
    from paper_2501_05244_b200.reconstruct import RsdEngine
    eng = RsdEngine(sl, grid)
    coeff = pf.phasor.device_coefficients(sl)
    eager = eng.run(coeff).clone()
    vol = torch.zeros_like(eager)
    for _ in range(3):
        eng.run_graphed(coeff, vol)
    torch.cuda.synchronize()
    assert torch.equal(vol, eager)
    assert eng.graph_kernels > 0


@pytest.mark.parametrize("n,nz,n_freq", [(64, 6, 5), (256, 4, 9), (512, 4, 32),
                                         (64, 5, 33), (64, 3, 64), (64, 4, 100),
                                         (128, 3, 400)])
def test_horner_phases_match_per_frequency_phases(rng, monkeypatch, n, nz, n_freq):
    """Kernel C with the illumination phase by Horner's rule over descending frequencies
    (pf_prop_rows_out_horner) = the ascending per-frequency phases (reference
    reconstruct.py:160-168), and both = the float64 oracle."""
    import importlib
    R = importlib.import_module("paper_2501_05244_b200.reconstruct")
    monkeypatch.setattr(R, "_FBATCH_BYTES", 0)
    p = 2.0 / n
    g = pf.UniformGrid2D(n, n, p, p, -1 + p / 2, -1 + p / 2, 0.0)
    sl = _random_slices(rng, pf.UniformRelay(g), n_freq=n_freq)
    grid = pf.CuboidGrid(pf.UniformGrid3D(n, n, nz, p, p, 0.4, g.x0, g.y0, 0.5))
    eng = R.RsdEngine(sl, grid)
    order, dk = eng.prop.freq_order(eng.freqs, 1)
    assert dk is not None and order[0] == n_freq - 1
    coeff = pf.phasor.device_coefficients(sl)
    hor = eng.run(coeff).clone()
    monkeypatch.setattr(R, "_HORNER", False)
    asc = eng.run(coeff)
    torch.cuda.synchronize()
    # z = exp(i dk d) is formed in float32 and raised to at most the 31st power (blocks of
    # 32 frequencies chained by a float64-reduced exp(i 32 dk d) beyond that): ~4e-6 at any
    # frequency count, 25x inside the 1e-4 gate
    assert O.rel_l2(hor.cpu().numpy(), asc.cpu().numpy()) < 1e-5
    if n <= 256:
        ref = O.rsd(sl, grid)
        assert O.rel_l2(hor.cpu().numpy().reshape(ref.shape), ref) < TOL
