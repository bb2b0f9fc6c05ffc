"""End-to-end physics checks of the reference acceptance suite, run on the GPU chain
simulate -> to_frequency -> rsd / light_transport_video (reference test_acceptance.py
sections 7 and 10)."""
import numpy as np
import pytest

import paper_2501_05244_b200 as pf
from paper_2501_05244_b200 import sim as S

pytestmark = pytest.mark.gpu


def _relay(n, pitch):
    o = -(n - 1) * pitch / 2
    return pf.UniformRelay(pf.UniformGrid2D(n, n, pitch, pitch, o, o, 0.0))


def _slices(scene, relay, ill, lambda_c, n_bins, delta_t=16e-12):
    m = S.simulate(scene, relay, ill, delta_t, n_bins)
    return pf.to_frequency(m, pf.build_kernel(lambda_c, n_bins, delta_t))


@pytest.mark.parametrize("z_true", [0.5, 1.0, 2.0])
def test_single_scatterer_localization(z_true):
    """Peak of |rsd| within max(2 cm, diffraction limit) laterally and max(dz, limit) in depth
    (reference test_acceptance.py:274-294)."""
    lambda_c = 0.04
    relay = _relay(32, 0.02)
    scene = S.Scene((S.Scatterer((0.01, 0.03, z_true)),))
    sl = _slices(scene, relay, pf.PointList(np.array([[0.0, 0.0]])), lambda_c, 1024)
    dz = 0.05
    grid = pf.CuboidGrid(pf.UniformGrid3D(9, 9, 9, 0.02, 0.02, dz, 0.01 - 4 * 0.02,
                                          0.03 - 4 * 0.02, z_true - 4 * dz))
    vol = pf.rsd(sl, grid)
    peak = grid.coordinates()[int(np.argmax(np.abs(vol.field)))]
    dx = pf.lateral_resolution(lambda_c, z_true, 32 * 0.02)
    assert np.hypot(peak[0] - 0.01, peak[1] - 0.03) <= max(0.02, dx)
    assert abs(peak[2] - z_true) <= max(dz, dx)


def test_video_time_zero_frame_is_bitwise_static():
    """reference test_acceptance.py:361-368."""
    relay = _relay(16, 0.02)
    scene = S.Scene((S.Scatterer((0.03, -0.02, 0.9), 1.0), S.Scatterer((-0.05, 0.04, 1.0), 0.7)))
    sl = _slices(scene, relay, pf.PointList(np.array([[0.0, 0.0]])), 0.06, 1024)
    grid = pf.CuboidGrid(pf.UniformGrid3D(8, 8, 2, 0.02, 0.02, 0.1, -0.07, -0.07, 0.9))
    static = pf.rsd(sl, grid)
    vid = pf.light_transport_video(sl, grid, np.array([0.0]))
    assert np.array_equal(vid.frame(0), static.frame(0))


def test_video_wavefront_arrival_at_one_meter():
    """The frame nearest the one-way flight time carries the peak (reference :370-385)."""
    depth = 1.0
    relay = _relay(16, 0.02)
    scene = S.Scene((S.Scatterer((0.01, 0.01, depth)),))
    sl = _slices(scene, relay, pf.PointList(np.array([[0.0, 0.0]])), 0.04, 2048)
    grid = pf.CuboidGrid(pf.UniformGrid3D(1, 1, 1, 0.02, 0.02, 0.05, 0.01, 0.01, depth))
    t_flight = depth / pf.SPEED_OF_LIGHT
    frame_dt = 50e-12
    times = t_flight + frame_dt * (np.arange(17) - 8)
    vid = pf.light_transport_video(sl, grid, times, include_illumination=False)
    peak = int(np.argmax(np.abs(vid.field[:, 0])))
    assert abs(times[peak] - t_flight) <= frame_dt
