"""On-chip propagation for the reference pad P = 140 (pf_prop_fbatch_onchip: every stage of
a (frequency, plane) unit in one CTA's shared memory), checked against the generic
shared-memory Stockham path (pf_prop_fbatch_generic, itself oracle-checked) on random
spectra and arbitrary crops, and against the oracle on config 1 (reference
reconstruct.py:372-383)."""

import numpy as np
import pytest
import torch

import paper_2501_05244_b200 as pf
from oracle import pf_oracle as O
from paper_2501_05244_b200 import _device as dev
import importlib

from paper_2501_05244_b200 import configs
from paper_2501_05244_b200.algorithms import Nursd1Engine

R = importlib.import_module("paper_2501_05244_b200.reconstruct")

pytestmark = pytest.mark.gpu


def _prop(nx, ny, nu0x, nu0y, include_illum, nplanes=5):
    zs = 0.6 + 0.13 * np.arange(nplanes)
    planes = [R.PlaneSpec(z - 0.01, 0.031, 0.029, -0.9, 0.031, -0.8, 0.029, z, 0, k)
              for k, z in enumerate(zs)]
    return R.Propagator(torch.device("cuda"), 140, 140, nx, ny, nu0x, nu0y, 1, include_illum,
                        planes, 140 * 140)


def _run(prop, uhat, freqs, ill, fw, onchip, groups=0):
    keep_oc, keep_g = prop.onchip, R._ONCHIP_GROUPS
    prop.onchip, R._ONCHIP_GROUPS = onchip, groups
    prop.__dict__.pop("_oc_key", None)
    try:
        g = prop.geom
        vol = torch.zeros(prop.nplanes * g.ny * g.nx, dtype=torch.complex64, device="cuda")
        prop.run_fbatch(uhat, 140 * 140, freqs, dev.ptr(ill), fw, vol)
        torch.cuda.synchronize()
        return vol.cpu().numpy()
    finally:
        prop.onchip, R._ONCHIP_GROUPS = keep_oc, keep_g


@pytest.mark.parametrize("nx,ny,nu0x,nu0y,illum", [
    (64, 64, -32, -32, True),      # config 1's centred crop
    (64, 64, -32, -32, False),
    (50, 37, -20, -9, True),       # ragged, off-centre
    (90, 100, -45, -50, True),     # the largest output plane the shared-memory budget takes
    (1, 1, 0, 0, True),            # one voxel
    (33, 70, 3, -69, True),        # crops that wrap the torus
])
@pytest.mark.parametrize("groups", [0, 1, 3])
def test_onchip_matches_generic(nx, ny, nu0x, nu0y, illum, groups):
    prop = _prop(nx, ny, nu0x, nu0y, illum)
    assert prop.onchip, "geometry should take the on-chip path"
    rng = np.random.default_rng(nx * 1000 + ny)
    nf = 7
    u = (rng.standard_normal((nf, 140, 140)) + 1j * rng.standard_normal((nf, 140, 140)))
    uhat = torch.from_numpy(u.astype(np.complex64).ravel()).cuda()
    freqs = 2 * np.pi * 3e8 / 0.06 * (1 + 0.05 * np.arange(nf))
    ill = torch.tensor([0.1, -0.2, 0.0], dtype=torch.float64, device="cuda")
    fw = torch.from_numpy(np.exp(1j * np.arange(nf) * 0.3).astype(np.complex64)).cuda()
    a = _run(prop, uhat, freqs, ill, fw, True, groups)
    b = _run(prop, uhat, freqs, ill, fw, False)
    assert O.rel_l2(a, b) < 2e-5, O.rel_l2(a, b)


def test_onchip_groups_bitwise_repeatable():
    prop = _prop(64, 64, -32, -32, True, nplanes=3)
    rng = np.random.default_rng(3)
    nf = 16
    u = rng.standard_normal((nf, 140, 140)) + 1j * rng.standard_normal((nf, 140, 140))
    uhat = torch.from_numpy(u.astype(np.complex64).ravel()).cuda()
    freqs = 2 * np.pi * 3e8 / 0.06 * (1 + 0.02 * np.arange(nf))
    ill = torch.tensor([0.0, 0.0, 0.0], dtype=torch.float64, device="cuda")
    fw = torch.ones(nf, dtype=torch.complex64, device="cuda")
    for groups in (1, 4, 16):
        a = _run(prop, uhat, freqs, ill, fw, True, groups)
        b = _run(prop, uhat, freqs, ill, fw, True, groups)
        assert np.array_equal(a, b)


def test_config1_onchip_vs_oracle_and_generic():
    cfg = configs.config(1)
    hist = configs.transients(cfg, device=torch.device("cuda"))
    k = pf.build_kernel(cfg.lambda_c, cfg.n_bins, cfg.delta_t)
    coeff = pf.to_frequency_device(hist, k, cfg.t0)
    sl = pf.DeviceFrequencySlices(k.frequencies, coeff, cfg.relay, cfg.illuminations)
    eng = Nursd1Engine(sl, cfg.grid)
    assert eng.prop.onchip and (eng.px, eng.py) == (140, 140)
    c = pf.phasor.device_coefficients(sl)
    v_on = eng.run(c).cpu().numpy().ravel()
    eng.prop.onchip = False
    v_gen = eng.run(c).cpu().numpy().ravel()
    ref = O.nursd1(sl.to_host(), cfg.grid).ravel()
    assert O.rel_l2(v_on, ref) < 1e-4
    assert O.rel_l2(v_on, v_gen) < 2e-5
    sh = cfg.grid.shape
    a = np.abs(v_on.reshape(sh)).max(axis=0)
    b = np.abs(ref.reshape(sh)).max(axis=0)
    assert np.argmax(a) == np.argmax(b)
