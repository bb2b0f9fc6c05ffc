"""Reference-compatible simulator against the reference's own output."""
import numpy as np
import pytest

import paper_2501_05244_b200 as pf
from paper_2501_05244_b200 import sim as S
from golden_io import load

pytestmark = pytest.mark.gpu


def _scene(d):
    return S.Scene(tuple(S.Scatterer(tuple(r[:3]), float(r[3])) for r in d["scatterers"]),
                   ambient=0.01)


def _setup():
    d = load("sim")
    relay = pf.UniformRelay(pf.UniformGrid2D(5, 4, 0.05, 0.06, -0.1, -0.09, 0.0))
    ill = pf.PointList(np.array([[0.0, 0.0], [0.05, -0.03]]))
    return d, relay, ill, _scene(d)


def test_simulate_matches_reference():
    d, relay, ill, scene = _setup()
    m = S.simulate(scene, relay, ill, 16e-12, 512, t0=2.5e-9)
    np.testing.assert_allclose(m.histograms, d["hist"], rtol=1e-12, atol=1e-12 * d["hist"].max())
    c = S.simulate(scene, relay, None, 16e-12, 512, t0=2.5e-9, confocal=True)
    np.testing.assert_allclose(c.histograms, d["hist_confocal"], rtol=1e-12,
                               atol=1e-12 * d["hist_confocal"].max())
    nf = S.simulate(scene, relay, ill, 16e-12, 512, t0=2.5e-9, falloff=False)
    np.testing.assert_allclose(nf.histograms, d["hist_nofalloff"], rtol=1e-12, atol=1e-12)
    # the seeded draw is the reference's numpy generator: identical counts
    noisy = S.add_poisson_noise(m, 50.0, seed=7)
    assert np.array_equal(noisy.histograms, d["hist_poisson"])


def test_simulate_errors_match_reference():
    d, relay, ill, scene = _setup()
    with pytest.raises(pf.ValidationError, match="outside the 64-bin window"):
        S.simulate(scene, relay, ill, 16e-12, 64, t0=2.5e-9)
    on_relay = S.Scene((S.Scatterer((-0.1, -0.09, 0.0)),))
    with pytest.raises(pf.ValidationError, match="coincides"):
        S.simulate(on_relay, relay, ill, 16e-12, 512)
    with pytest.raises(pf.ValidationError, match="explicit illumination"):
        S.simulate(scene, relay, None, 16e-12, 512)
