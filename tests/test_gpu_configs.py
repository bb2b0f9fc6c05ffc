"""BASELINE configurations at full size on the GPU, checked against the CPU oracle.

Configs 0 and 1 are compared over the whole volume; configs 3 and 4 over depth-plane
subsets with every frequency (each (frequency, plane) unit is independent, so a plane
subset is an exact slice of the full computation).  The slices fed to the oracle are the
GPU's K1 output (checked separately against the oracle's to_frequency on a trace subset).
"""

import json
import os

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


def _check(vol_field, ref, shape, name=None):
    """North-star gates: relative L2 and the project_max_depth argmax, with the
    reference image's top-2 gap reported (near-ties); one JSON line
    per check goes to $PF_PARITY_LOG when set."""
    rel = O.rel_l2(vol_field, ref)
    a = np.abs(vol_field.reshape(shape)).max(axis=0).ravel()
    b = np.abs(ref.reshape(shape)).max(axis=0).ravel()
    top2 = np.sort(b)[-2:]
    gap = float((top2[1] - top2[0]) / top2[1])
    same = int(np.argmax(a)) == int(np.argmax(b))
    log = os.environ.get("PF_PARITY_LOG")
    if log:
        with open(log, "a") as f:
            f.write(json.dumps({"case": name or os.environ.get("PYTEST_CURRENT_TEST", "?"),
                                "rel_l2": rel, "argmax_same": same, "top2_gap": gap,
                                "shape": list(shape)}) + "\n")
    assert rel < TOL
    assert same, f"argmax differs (reference top-2 gap {gap:.3e})"


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


@pytest.mark.parametrize("planes", [(0, 2), (200, 202)])
def test_config4_nursd1_on_lattice_equals_zero_filled_rsd(planes):
    """SURVEY 8(d) "c4 NURSD1": 131,072 on-lattice nodes; nursd1 == rsd on the zero-filled
    lattice (F4), and both match the float64 oracle rsd."""
    cfg = configs.config(5)
    sl, k = _slices(cfg)
    eng = Nursd1Engine(sl, cfg.grid, plane_range=planes)
    assert eng.px == 1024 and eng.prop.transposed        # pad-free on lattice -> register path
    vol = eng.run(sl.device_coefficients)[0].cpu().numpy()
    base = configs.config(4)
    full = np.zeros((k.n_freq, 1, base.relay.count), dtype=np.complex64)
    full[:, :, cfg.lattice_nodes] = sl.device_coefficients.cpu().numpy()
    zf = pf.DeviceFrequencySlices(k.frequencies, torch.from_numpy(full).cuda(), base.relay,
                                  base.illuminations)
    vr = RsdEngine(zf, base.grid, plane_range=planes).run(zf.device_coefficients)[0]
    assert O.rel_l2(vol, vr.cpu().numpy()) < 1e-5
    ref = O.rsd(zf.to_host(), base.grid, plane_range=planes)
    _check(vol, ref, (planes[1] - planes[0], 512, 512))


def test_config4_full_size_linearity_and_frequency_additivity():
    """Full config-4 volume (67 M voxels, all 256 planes, 32 frequencies): size-independent
    properties of the reference operator. (1) Linearity in the wavefront:
    V(a u1 + b u2) = a V(u1) + b V(u2). (2) The volume is the ascending-frequency sum
    (reconstruct.py:163-177): V(all f) = V(f < 16) + V(f >= 16)."""
    cfg = configs.config(4)
    sl, k = _slices(cfg)
    c = sl.device_coefficients
    g = torch.Generator(device="cuda").manual_seed(3)
    u2 = torch.randn(c.shape, dtype=torch.complex64, device="cuda", generator=g)
    eng = RsdEngine(sl, cfg.grid)
    a, b = 0.7 - 0.2j, -1.3 + 0.5j
    v1 = eng.run(c).clone()
    v2 = eng.run(u2).clone()
    v12 = eng.run((a * c + b * u2).contiguous()).clone()
    lin = ((v12 - (a * v1 + b * v2)).norm() / v12.norm()).item()
    assert lin < 1e-5, lin
    lo = c.clone()
    lo[16:] = 0
    hi = c - lo
    vlo = eng.run(lo).clone()
    vhi = eng.run(hi)
    add = ((v1 - (vlo + vhi)).norm() / v1.norm()).item()
    assert add < 1e-6, add


def test_config5_full_size_nursd1_equals_zero_filled_rsd():
    """All 256 planes of the c4-NURSD1 workload: nursd1 on the 131,072 lattice nodes equals rsd
    on the zero-filled 512x512 lattice over the whole 67 M-voxel volume."""
    cfg = configs.config(5)
    sl, k = _slices(cfg)
    vol = Nursd1Engine(sl, cfg.grid).run(sl.device_coefficients).clone()
    base = configs.config(4)
    full = torch.zeros((k.n_freq, 1, base.relay.count), dtype=torch.complex64, device="cuda")
    full[:, :, torch.from_numpy(cfg.lattice_nodes).cuda()] = sl.device_coefficients
    zf = pf.DeviceFrequencySlices(k.frequencies, full, base.relay, base.illuminations)
    vr = RsdEngine(zf, base.grid).run(full)
    assert ((vol - vr).norm() / vr.norm()).item() < 1e-5


def test_config3_full_size_linearity():
    """srsd over all 128 frustum planes (8.4 M voxels): V(a u1 + b u2) = a V(u1) + b V(u2)."""
    cfg = configs.config(3)
    sl, k = _slices(cfg)
    c = sl.device_coefficients
    g = torch.Generator(device="cuda").manual_seed(5)
    u2 = torch.randn(c.shape, dtype=torch.complex64, device="cuda", generator=g)
    eng = SrsdEngine(sl, cfg.grid)
    a, b = 1.1 + 0.4j, -0.6 - 0.9j
    v1 = eng.run(c).clone()
    v2 = eng.run(u2).clone()
    v12 = eng.run((a * c + b * u2).contiguous())
    assert ((v12 - (a * v1 + b * v2)).norm() / v12.norm()).item() < 1e-5
