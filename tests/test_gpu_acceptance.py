"""The reference acceptance suite's oracle-consistency scenes on the GPU.

Reference tests/test_acceptance.py:204-266 draws 20 scenes (seeds 6000+i) that cycle
through all eight algorithms with one or two illuminations and scatterers, and requires
the normalised cross-correlation of |field| with the phase-only backprojection oracle
(reference oracle.py:86-117) to reach 0.95 (0.9 for the 3D relays).  The fixtures
(tests/golden/acc_*.npz) hold the reference's own reconstruction and backprojection of
each scene; the GPU must match the reconstruction to the north-star tolerance and clear
the same NCC floor.
"""
import numpy as np
import pytest

import paper_2501_05244_b200 as pf
from oracle import pf_oracle as O
from golden_io import grid_from, load, slices_from

pytestmark = pytest.mark.gpu
TOL = 1e-4


def _ncc(a, b):
    """Pearson correlation of magnitudes (reference metrics.py:90-100)."""
    x = np.abs(a).ravel() - np.abs(a).mean()
    y = np.abs(b).ravel() - np.abs(b).mean()
    return float(np.sum(x * y) / (np.linalg.norm(x) * np.linalg.norm(y)))


@pytest.mark.parametrize("i", range(20))
def test_acceptance_scene(i):
    d = load(f"acc_{i}")
    sl, grid = slices_from(d), grid_from(d)
    algo = str(d["algo"])
    opts = {} if np.isnan(float(d["alpha"])) else {"alpha": float(d["alpha"])}
    vol = pf.reconstruct(sl, grid, algo, **opts)
    assert O.rel_l2(vol.field, d["field"]) < TOL, (algo, O.rel_l2(vol.field, d["field"]))
    score = _ncc(vol.field, d["backproject"])
    assert score >= float(d["floor"]), (algo, score)
