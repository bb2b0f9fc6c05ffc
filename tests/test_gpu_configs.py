"""BASELINE configurations at full size on the GPU, checked against the CPU oracle.

Configs 0 and 1 are compared over the whole volume; configs 3 and 4 over depth-plane
subsets with every frequency (each (frequency, plane) unit is independent, so a plane
subset is an exact slice of the full computation).  The slices fed to the oracle are the
GPU's K1 output (checked separately against the oracle's to_frequency on a trace subset).
"""

import numpy as np
import pytest
import torch

import paper_2501_05244_b200 as pf
from oracle import pf_oracle as O
from paper_2501_05244_b200 import configs
from paper_2501_05244_b200.algorithms import Nursd1Engine, SrsdEngine
from paper_2501_05244_b200.reconstruct import RsdEngine

pytestmark = pytest.mark.gpu
TOL = 1e-4


def _slices(cfg):
    hist = configs.transients(cfg, device=torch.device("cuda"))
    k = pf.build_kernel(cfg.lambda_c, cfg.n_bins, cfg.delta_t)
    coeff = pf.to_frequency_device(hist, k, cfg.t0)
    sl = pf.DeviceFrequencySlices(k.frequencies, coeff, cfg.relay, cfg.illuminations)
    # K1 parity on a trace subset (float32 input, float64 oracle)
    h = hist[0, :2048].cpu().numpy().astype(np.float64)
    ref = O.to_frequency(h, k.bin_indices, k.frequencies, k.weights, cfg.t0)
    got = coeff[:, 0, :2048].cpu().numpy().T
    assert O.rel_l2(got, ref) < 1e-6
    return sl, k


def _check(vol_field, ref, shape):
    assert O.rel_l2(vol_field, ref) < TOL
    a = np.abs(vol_field.reshape(shape)).max(axis=0)
    b = np.abs(ref.reshape(shape)).max(axis=0)
    assert int(np.argmax(a)) == int(np.argmax(b))


def test_config0_rsd_full():
    cfg = configs.config(0)
    sl, k = _slices(cfg)
    assert k.n_freq == 16
    vol = pf.rsd(sl, cfg.grid)
    _check(vol.field, O.rsd(sl.to_host(), cfg.grid), cfg.grid.shape)


def test_config1_nursd1_full():
    cfg = configs.config(1)
    sl, k = _slices(cfg)
    eng = Nursd1Engine(sl, cfg.grid)
    assert (eng.px, eng.py) == (140, 140)          # reference pad rule
    vol = pf.nursd1(sl, cfg.grid)
    _check(vol.field, O.nursd1(sl.to_host(), cfg.grid), cfg.grid.shape)


@pytest.mark.parametrize("planes", [(0, 2), (70, 72), (126, 128)])
def test_config3_srsd_plane_subsets(planes):
    cfg = configs.config(3)
    sl, k = _slices(cfg)
    assert k.n_freq == 24
    eng = SrsdEngine(sl, cfg.grid, plane_range=planes)
    assert eng.px == 512                            # next_fast_len(2N)
    vol = eng.run(sl.device_coefficients)[0].cpu().numpy()
    ref = O.srsd(sl.to_host(), cfg.grid, plane_range=planes)
    _check(vol, ref, (planes[1] - planes[0], 256, 256))


@pytest.mark.parametrize("planes", [(0, 2), (128, 130)])
def test_config4_rsd_plane_subsets(planes):
    cfg = configs.config(4)
    sl, k = _slices(cfg)
    assert k.n_freq == 32
    eng = RsdEngine(sl, cfg.grid, plane_range=planes)
    assert eng.px == 1024
    vol = eng.run(sl.device_coefficients)[0].cpu().numpy()
    ref = O.rsd(sl.to_host(), cfg.grid, plane_range=planes)
    _check(vol, ref, (2, 512, 512))


def test_config4_plane_subset_equals_full_run_slice():
    """Plane sharding is exact: a shard's planes are bitwise the full run's planes."""
    cfg = configs.config(4)
    sl, _ = _slices(cfg)
    full = RsdEngine(sl, cfg.grid).run(sl.device_coefficients)
    part = RsdEngine(sl, cfg.grid, plane_range=(64, 96)).run(sl.device_coefficients)
    pv = 512 * 512
    assert torch.equal(full[0, 64 * pv:96 * pv], part[0])
