"""Pin the CPU oracle against golden vectors produced by the reference itself."""

import numpy as np
import pytest

from oracle import pf_oracle as O
from golden_io import REC_CASES, case_call, grid_from, load, slices_from

ORACLE_FN = {"rsd": O.rsd, "srsd": O.srsd, "nursd1": O.nursd1, "nursd2": O.nursd2,
             "nursd3": O.nursd3, "srsd-nursd2": O.srsd_nursd2, "nursd3d": O.nursd3d,
             "rsd3d": O.rsd3d}


def test_build_kernel_kats():
    d = load("phasor")
    # reference test_phasor.py:29-30
    b, _, _ = O.build_kernel(0.04, 4096, 16e-12)
    assert b.size == 95
    for i in range(int(d["n_kats"])):
        lam, nb, dt = d[f"k{i}_args"]
        b, f, w = O.build_kernel(lam, int(nb), dt)
        assert np.array_equal(b, d[f"k{i}_bins"])
        assert np.allclose(f, d[f"k{i}_freqs"], rtol=1e-15)
        assert np.allclose(w, d[f"k{i}_weights"], rtol=1e-13)


def test_to_frequency_golden():
    d = load("phasor")
    for i in range(int(d["n_tf"])):
        nb, dt, t0, lam = d[f"tf{i}_args"]
        b, f, w = O.build_kernel(lam, int(nb), dt)
        got = O.to_frequency(d[f"tf{i}_hist"], b, f, w, t0)
        assert O.rel_linf(got, d[f"tf{i}_coeff"]) < 1e-12
        direct = O.to_frequency_direct(d[f"tf{i}_hist"], b, f, w, t0, dt)
        assert O.rel_linf(got, direct) < 1e-10


def test_spectral_golden():
    d = load("spectral")
    for i in range(int(d["n_c"])):
        assert O.rel_linf(O.cfft2(d[f"c{i}_u"]), d[f"c{i}_fwd"]) < 1e-13
        assert O.rel_linf(O.cifft2(d[f"c{i}_u"]), d[f"c{i}_inv"]) < 1e-13
    for i in range(int(d["n_s"])):
        m, a, o = d[f"s{i}_args"]
        got = O.sfft_1d(d[f"s{i}_u"], a, int(o))
        assert O.rel_linf(got, d[f"s{i}_out"]) < 1e-12
        assert O.rel_linf(got, d[f"s{i}_slow"]) < 1e-9
    assert O.rel_linf(O.sfft_2d_centered(d["s2d_u"], 0.45, 0.8), d["s2d_out"]) < 1e-12
    for i in range(int(d["n_n"])):
        modes = tuple(int(m) for m in d[f"n{i}_modes"])
        eps = float(d[f"n{i}_eps"])
        t1 = O.nufft1(d[f"n{i}_pts"], d[f"n{i}_vals"], modes, eps)
        t2 = O.nufft2(d[f"n{i}_coeff"], d[f"n{i}_pts"], eps)
        assert O.rel_linf(t1, d[f"n{i}_t1"]) < 1e-12
        assert O.rel_linf(t2, d[f"n{i}_t2"]) < 1e-12
        assert O.rel_linf(t1, d[f"n{i}_d1"]) < max(eps, 1e-12) * 10


@pytest.mark.parametrize("name", REC_CASES)
def test_reconstruction_golden(name):
    d = load(f"rec_{name}")
    sl, grid = slices_from(d), grid_from(d)
    alg, kw = case_call(name)
    kw = dict(kw)
    if kw.get("times") == "times":
        kw["times"] = d["times"]
    if alg == "rsd" and "padding" not in kw:
        kw["padding"] = "exact"
    got = ORACLE_FN[alg](sl, grid, **kw)
    assert O.rel_linf(got, d["field"]) < 1e-11, name
    if "literal" in d:
        assert O.rel_linf(got, d["literal"]) < 1e-10
    if "video" in d:
        vid = ORACLE_FN[alg](sl, grid, times=np.array([0.0, 5e-10]))
        assert O.rel_linf(vid, d["video"]) < 1e-11


@pytest.mark.parametrize("i", range(20))
def test_oracle_on_acceptance_scenes(i):
    """The oracle reproduces the reference on its acceptance-suite scenes (all eight
    algorithm paths, reference test_acceptance.py:204-266)."""
    d = load(f"acc_{i}")
    algo = str(d["algo"])
    kw = {} if np.isnan(float(d["alpha"])) else {"alpha": float(d["alpha"])}
    got = ORACLE_FN[algo](slices_from(d), grid_from(d), **kw)
    assert O.rel_linf(got, d["field"]) < 1e-9, algo
